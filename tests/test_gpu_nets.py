"""GPU parity for the paper's own 2-D workloads (DESIGN.md
reading #16): Figure 4's 224x224 image through three 32->32 layers of 4x4
kernels with F(5,4) (Table 1 (c), D = 8) and F(3,4), and
Figure 3's single 4x4 layer on a 1024x1024 image, all at the
full spatial size, batch 1, against the float64 direct oracle.

Tolerance (reading #16): oracle.fp32model's float32 / 3xTF32 model
run through the same chain of layers on the same inputs (each layer's
float32 output feeding the next, as on the device); the GPU must stay within
K_REL = 4x the model's relL2 and K_MAX = 8x its max-abs / max|y| against the
float64 chain.
"""
import numpy as np
import pytest
import torch

import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.workloads import NETS, make_net_inputs
from oracle import direct, fp32model as fm

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.cuda.set_device(0)


def _net(net_cfg, B):
    layers = [(l.N, l.dims, l.m, l.r, l.C, l.K, l.padding) for l in net_cfg.layers]
    return pkg.Net(layers, B)


def _model_chain(layers, x, gs, relu=False):
    """The chain in the float32 model (layer outputs rounded to float32 and fed on)."""
    y = x
    for l, g in zip(layers, gs):
        y = fm.winograd_model(y, g, l.pad, l.m, l.r)
        if relu:
            y = np.maximum(y, 0).astype(np.float32)
    return y


def _tol(layers, x, gs, ref, relu=False):
    rel, mx = fm.errors(_model_chain(layers, x, gs, relu), ref)
    return fm.K_REL * rel, fm.K_MAX * mx


@pytest.mark.parametrize("name", ["fig4_f54", "fig4_f34"])
def test_fig4_chain_full_size(name):
    cfg = NETS[name]
    x, gs = make_net_inputs(cfg, seed=0, batch=1)
    net = _net(cfg, 1)
    net.filter_transform([g.cuda() for g in gs])
    y = net.forward(x.cuda()).cpu().double().numpy()
    net.close()
    ref = x.double().numpy()
    for g in gs:     # each layer in float64 (the oracle rounds its input activations to fp32)
        ref = direct.direct_conv_f64(ref, g.double().numpy(), 0)
    assert y.shape == ref.shape == (1, 32, 215, 215)
    rel, mx = fm.errors(y, ref)
    tl, tm = _tol(cfg.layers, x.numpy(), [g.numpy() for g in gs], ref)
    print("%s relL2=%.2e max=%.2e tol=%.1e/%.1e" % (name, rel, mx, tl, tm))
    assert rel <= tl and mx <= tm


def test_fig3_layer_sampled():
    cfg = NETS["fig3_f54"]
    x, gs = make_net_inputs(cfg, seed=0, batch=1)
    net = _net(cfg, 1)
    net.filter_transform([g.cuda() for g in gs])
    y = net.forward(x.cuda()).cpu().double().numpy()
    net.close()
    assert y.shape == (1, 32, 1021, 1021)
    rng = np.random.default_rng(1)
    idx = rng.integers(0, y.size, 20000)
    idx[:4] = [0, y.size - 1, 1020, 1021 * 1021 - 1]          # corners of the first plane, last output
    ref = direct.direct_conv_at(x.numpy(), gs[0].numpy(), 0, idx)
    got = y.reshape(-1)[idx]
    rel, mx = fm.errors(got, ref)
    # model bound on the top-left 256 x 256 of the same image (same statistics)
    xs = x.numpy()[:, :, :256, :256]
    l0 = cfg.layers[0]
    refs = direct.direct_conv_f64(xs, gs[0].numpy(), 0)
    tl, tm = _tol([l0], xs, [gs[0].numpy()], refs)
    print("fig3 sampled relL2=%.2e max=%.2e tol=%.1e/%.1e" % (rel, mx, tl, tm))
    assert rel <= tl and mx <= tm


def test_chain_relu_and_batch():
    # a reduced Figure-4 chain at batch 3 with f = ReLU after every layer
    cfg = NETS["fig4_f34"]
    from dataclasses import replace
    dims = [41, 37]
    layers = []
    for l in cfg.layers:
        layers.append(replace(l, dims=tuple(dims)))
        dims = [d - l.r + 1 for d in dims]
    small = replace(cfg, layers=tuple(layers))
    x, gs = make_net_inputs(small, seed=3, batch=3)
    net = _net(small, 3)
    net.filter_transform([g.cuda() for g in gs])
    y = net.forward(x.cuda(), relu=True).cpu().double().numpy()
    net.close()
    ref = x.double().numpy()
    for g in gs:
        ref = np.maximum(direct.direct_conv_f64(ref, g.double().numpy(), 0), 0.0)
    rel, mx = fm.errors(y, ref)
    tl, tm = _tol(small.layers, x.numpy(), [g.numpy() for g in gs], ref, relu=True)
    assert rel <= tl and mx <= tm, (rel, mx, tl, tm)
    assert (y >= 0).all()


def test_chain_shape_mismatch_is_an_error():
    with pytest.raises(ValueError):
        pkg.Net([(2, (16, 16), 3, 4, 8, 8, (0, 0)), (2, (16, 16), 3, 4, 8, 8, (0, 0))], 1)


def test_chain_graph_replay_matches_eager():
    cfg = NETS["fig4_f34"]
    x, gs = make_net_inputs(cfg, seed=4, batch=1)
    net = _net(cfg, 1)
    net.filter_transform([g.cuda() for g in gs])
    xd = x.cuda()
    y_eager = net.forward(xd).clone()
    replay = net.capture(xd)
    y_graph = replay()
    torch.cuda.synchronize()
    assert torch.equal(y_graph, y_eager)
    xd.mul_(0.5)                                   # same memory, new values: the graph sees them
    y2 = replay().clone()
    assert torch.equal(y2, net.forward(xd))
    net.close()
