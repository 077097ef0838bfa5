"""A chain of N-D Winograd layers on one GPU (the paper's three-layer pass of
Figure 4).

Each layer is a `Plan`; the output tensor of layer l ([B][K][out..], NCHW) is
the input tensor of layer l+1 as it stands, so there is no inter-layer
"reshuffling" kernel (the paper counts it in its timings): the
input transform of the next layer reads the previous output directly.  All
arithmetic runs in the plans' kernels; this module only allocates the
activations and orders the launches on one stream.
"""
from __future__ import annotations

from typing import Optional, Sequence

from .wino import Plan


class Net:
    """Net(layers, batch, points=None, device=-1): `layers` is a sequence of
    (N, dims, m, r, C, K, padding) tuples; layer l+1's dims and C must be
    layer l's output dims and K."""

    def __init__(self, layers: Sequence[tuple], batch: int, points: Optional[str] = None, device: int = -1):
        import torch
        self.plans = []
        prev = None
        for (N, dims, m, r, C, K, padding) in layers:
            if prev is not None and (tuple(prev.out_dims) != tuple(dims) or prev.K != C):
                raise ValueError("layer %d input (%s, C=%d) does not match the previous output (%s, K=%d)"
                                 % (len(self.plans), tuple(dims), C, tuple(prev.out_dims), prev.K))
            prev = Plan(N, dims, m, r, C, K, batch, padding, points=points, device=device)
            self.plans.append(prev)
        self.batch = batch
        dev = torch.device("cuda", device if device >= 0 else torch.cuda.current_device())
        # activations between layers stay in HBM; the last one is the result
        self.acts = [torch.empty((batch, p.K) + tuple(p.out_dims), device=dev, dtype=torch.float32)
                     for p in self.plans]

    def filter_transform(self, gs, stream=None) -> None:
        if len(gs) != len(self.plans):
            raise ValueError("expected %d kernel tensors, got %d" % (len(self.plans), len(gs)))
        for p, g in zip(self.plans, gs):
            p.filter_transform(g, stream)

    def forward(self, x, stream=None, relu: bool = False):
        """y_L = conv_L(... conv_1(x)); with relu=True every layer applies
        f = ReLU (Eq. (2)) in its output-transform epilogue.  Returns the last
        activation (a tensor owned by the Net, overwritten by the next call)."""
        if x.shape[0] != self.batch:
            raise ValueError("batch %d != planned %d" % (x.shape[0], self.batch))
        h = x
        for p, y in zip(self.plans, self.acts):
            p.forward(h, y, stream, relu=relu)
            h = y
        return h

    def capture(self, x, relu: bool = False):
        """Record one forward on the device tensor `x` into a CUDA graph and
        return a function that replays it (same x memory, result in the Net's
        last activation).  For launch-bound small batches: one graph launch
        replaces the 3 kernel launches per layer (measured: Figure 4 at batch
        1, 0.106 -> 0.094 ms with F(5,4), 0.142 -> 0.107 ms with F(3,4))."""
        import torch
        if x.shape[0] != self.batch:
            raise ValueError("batch %d != planned %d" % (x.shape[0], self.batch))
        s = torch.cuda.Stream(device=x.device)
        s.wait_stream(torch.cuda.current_stream(x.device))
        with torch.cuda.stream(s):
            self.forward(x, s, relu)            # warm-up outside the capture
        s.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            self.forward(x, s, relu)

        def replay():
            graph.replay()
            return self.acts[-1]
        replay.graph = graph
        return replay

    def close(self) -> None:
        for p in self.plans:
            p.close()
        self.plans = []
