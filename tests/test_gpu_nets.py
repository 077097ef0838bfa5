"""GPU parity for the paper's own 2-D workloads (DESIGN.md
reading #16): Figure 4's 224x224 image through three 32->32 layers of 4x4
kernels with F(5,4) (Table 1 (c), D = 8) and F(3,4), and
Figure 3's single 4x4 layer on a 1024x1024 image, all at the
full spatial size, batch 1, against the float64 direct oracle.

Tolerance: the per-layer bound of the arbitrary-(m, r) tests (reading #15,
relL2 <= 4e-7 * c_alpha^2, c_8 = 5, c_6 = 2.2) times the number of layers
(each layer's relative error passes through the later, norm-preserving He
layers and adds); max-abs <= 10x that, relative to max|y|.
"""
import numpy as np
import pytest
import torch

import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.workloads import NETS, make_net_inputs
from oracle import direct

pytestmark = pytest.mark.gpu

GROWTH = {6: 2.2, 8: 5.0}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.cuda.set_device(0)


def _net(net_cfg, B):
    layers = [(l.N, l.dims, l.m, l.r, l.C, l.K, l.padding) for l in net_cfg.layers]
    return pkg.Net(layers, B)


def _tol(net_cfg):
    l0 = net_cfg.layers[0]
    return len(net_cfg.layers) * 4e-7 * GROWTH[l0.alpha] ** l0.N


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
    rel = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    mx = np.abs(y - ref).max() / np.abs(ref).max()
    tol = _tol(cfg)
    print("%s relL2=%.2e max=%.2e tol=%.1e" % (name, rel, mx, tol))
    assert rel <= tol and mx <= 10 * tol


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
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    tol = _tol(cfg)
    print("fig3 sampled relL2=%.2e tol=%.1e" % (rel, tol))
    assert rel <= tol and np.abs(got - ref).max() <= 10 * tol * np.abs(ref).max()


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
    rel = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    assert rel <= _tol(small), rel
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
