"""GPU parity of the CUDA path against the CPU oracle (run on a B200: -m gpu).

Every comparison calls the product through the C ABI (paper_1611_06565_b200.wino)
and compares with oracle/ on the same seeded inputs (workloads.make_inputs):

* shrunken configs (ragged extents, several 128-row GEMM blocks with a partial
  last one, C/K not multiples of the tile widths): every output element vs the
  float64 direct correlation (oracle.direct), both GEMM schemes;
* full BASELINE.json configs, in bench.py's launch configuration: 4096 sampled
  outputs computed one by one by the oracle (c1, c2: every element);
* stage parity (U, V, M) vs the step-by-step float64 oracle (oracle.winograd);
* properties: determinism, batch independence, filter-cache idempotence,
  zero input, error codes, host-buffer entry point.

Tolerances are BASELINE.json north_star's: relL2 <= 2e-6 and max <= 1e-4 max|y|
for F(2^N,3^N); 1e-5 and 1e-3 for F(4^N,3^N).
"""
import numpy as np
import pytest
import torch

import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200 import wino
from paper_1611_06565_b200.workloads import CONFIGS, SMALL, make_inputs, tolerance
from oracle import direct, toomcook as tc, winograd as wg

pytestmark = pytest.mark.gpu

DEFAULT_POINTS = {4: "0,1,-1,inf", 6: "0,3/2,-3/2,2/3,-2/3,inf"}   # DESIGN.md reading #5


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.cuda.set_device(0)


def run(cfg, gemm_mode=0, points=None, batch=None, plan_batch=None, fuse=0):
    x, g = make_inputs(cfg, batch=batch)
    plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, plan_batch or x.shape[0], cfg.padding,
                    points=points, gemm_mode=gemm_mode, fuse=fuse)
    plan.filter_transform(g.cuda())
    y = plan.forward(x.cuda())
    torch.cuda.synchronize()
    return x, g, y.cpu(), plan


def errs(y, ref):
    y = np.asarray(y, dtype=np.float64)
    rel = float(np.linalg.norm(y - ref) / np.linalg.norm(ref))
    mx = float(np.abs(y - ref).max() / np.abs(ref).max())
    return rel, mx


@pytest.mark.parametrize("gemm_mode", [wino.WINO_GEMM_3XTF32, wino.WINO_GEMM_FFMA])
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_small_full_parity(name, gemm_mode):
    cfg = SMALL[name]
    x, g, y, plan = run(cfg, gemm_mode)
    ref = direct.direct_conv_f64(x.numpy(), g.numpy(), cfg.pad)
    assert y.shape == ref.shape
    rel, mx = errs(y.numpy(), ref)
    tl, tm = tolerance(cfg)
    print("%s mode=%d relL2=%.3e max=%.3e" % (cfg.name, gemm_mode, rel, mx))
    assert rel <= tl and mx <= tm
    plan.close()


def winograd_f64_full(cfg, x, g):
    """Every output of the full config in float64 by oracle.winograd (Eq. (3)-(5)
    step by step; pinned to the direct oracle at 1e-12 in
    tests/test_oracle_winograd.py), one sample at a time to bound host memory."""
    A, B, C = tc.synthesize(cfg.m, cfg.r, DEFAULT_POINTS[cfg.alpha])
    xn, gn = x.numpy().astype(np.float64), g.numpy().astype(np.float64)
    out = np.empty((cfg.batch, cfg.K) + cfg.out_dims, dtype=np.float64)
    for b in range(cfg.batch):
        out[b:b + 1] = wg.winograd_nd(xn[b:b + 1], gn, cfg.padding, A, B, C, exact=False)[0]
    return out


FULL_SIZE_ERRORS = {}


def _record_error(name, cfg, rel, mx, n):
    # the achieved error per (N, m) at full size (BASELINE.json north_star asks
    # for it to be reported): appended to gpurun_out/parity_full_size.json
    import json
    import os
    path = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "parity_full_size.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    try:
        with open(path) as f:
            d = json.load(f)
    except (OSError, ValueError):
        d = {}
    d[name] = {"N": cfg.N, "m": cfg.m, "F": "F(%d^%d,%d^%d)" % (cfg.m, cfg.N, cfg.r, cfg.N), "outputs": n,
               "relL2": rel, "max_over_maxy": mx, "tol": list(tolerance(cfg))}
    with open(path, "w") as f:
        json.dump(d, f, indent=1)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_full_size(name):
    """BASELINE.json configs at full size in bench.py's launch configuration.
    c1, c2: every output vs the direct oracle; c3-c5: every output vs the
    float64 Winograd oracle, plus 4224 outputs vs the direct oracle."""
    cfg = CONFIGS[name]
    x, g, y, plan = run(cfg)
    plan.close()
    tl, tm = tolerance(cfg)
    if name in ("c1", "c2"):
        ref = direct.direct_conv_f64(x.numpy(), g.numpy(), cfg.pad)
        rel, mx = errs(y.numpy(), ref)
    else:
        ref = winograd_f64_full(cfg, x, g)
        rel, mx = errs(y.numpy(), ref)
        rng = np.random.default_rng(1234)
        n = y.numel()
        # random outputs plus the first/last elements (edge tiles, first/last batch, k)
        idx = np.unique(np.concatenate([rng.integers(0, n, 4096), np.arange(64), np.arange(n - 64, n)]))
        refd = direct.direct_conv_at(x.numpy(), g.numpy(), cfg.pad, idx)
        assert np.abs(ref.reshape(-1)[idx] - refd).max() <= 1e-11 * np.abs(refd).max()
        rs, ms = errs(y.numpy().reshape(-1)[idx], refd)
        assert rs <= tl and ms <= tm
    FULL_SIZE_ERRORS[name] = (rel, mx)
    _record_error(name, cfg, rel, mx, y.numel())
    print("%s full (%d outputs) relL2=%.3e max=%.3e (tol %.0e/%.0e)" % (name, y.numel(), rel, mx, tl, tm))
    assert rel <= tl and mx <= tm


def _oracle_stages(cfg, x, g, T):
    A, B, C = tc.synthesize(cfg.m, cfg.r, DEFAULT_POINTS[cfg.alpha])
    y, st = wg.winograd_nd(x.numpy().astype(np.float64), g.numpy().astype(np.float64), cfg.padding,
                           A, B, C, exact=False)
    return st


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_stage_parity(name, monkeypatch):
    # the unfused pipeline's workspace (V, M); the folded GEMM's W is checked
    # in tests/test_gpu_fold.py
    monkeypatch.setenv("WINO_FOLD", "0")
    cfg = SMALL[name]
    x, g, y, plan = run(cfg)
    info = plan.info
    T = cfg.tiles()
    P, Ts, Ks = info["n_points"], info["T_stride"], info["K_stride"]
    st = _oracle_stages(cfg, x, g, T)
    # U (a1): U_hi + U_lo vs G_hat [P][C][K]
    u = plan.filter_tensor().cpu().double().numpy()
    n = P * cfg.C * Ks
    U = (u[:n] + u[n:2 * n]).reshape(P, cfg.C, Ks)[:, :, :cfg.K]
    Uref = st["U"]
    assert np.abs(U - Uref).max() <= 1e-6 * np.abs(Uref).max()
    # V (a2): [P][C][T_s] vs D_hat [P][T][C]
    V, M = plan.workspace()
    Vg = V.cpu().double().numpy()
    Vref = st["V"].transpose(0, 2, 1)
    assert np.all(Vg[:, :, T:] == 0.0), "padding rows of V must be zero"
    Vg = Vg[:, :, :T]
    assert np.linalg.norm(Vg - Vref) / np.linalg.norm(Vref) <= 1e-6
    # M (a3): [P][K][T_s] vs S_hat [P][T][K]
    Mg = M.cpu().double().numpy()[:, :, :T]
    Mref = st["Shat"].transpose(0, 2, 1)
    rel = np.linalg.norm(Mg - Mref) / np.linalg.norm(Mref)
    print("%s stage M relL2 %.3e" % (name, rel))
    assert rel <= tolerance(cfg)[0]
    plan.close()


def test_one_tf32_is_not_enough():
    # the single-product tf32 GEMM misses the fp32 tolerance by orders of magnitude
    # (reading #7): evidence the 3xTF32 split is required and active.
    cfg = SMALL["c2"]
    x, g, y, plan = run(cfg, wino.WINO_GEMM_1XTF32)
    rel, _ = errs(y.numpy(), direct.direct_conv_f64(x.numpy(), g.numpy(), cfg.pad))
    assert 1e-5 < rel < 1e-2
    plan.close()


@pytest.mark.parametrize("points", ["0,1,-1,2,-2,inf", "0,1,-1,1/2,-1/2,inf", "0,-1,1,2/3,-2/3,inf"])
def test_custom_points(points):
    cfg = SMALL["c2"]
    x, g, y, plan = run(cfg, points=points)
    rel, mx = errs(y.numpy(), direct.direct_conv_f64(x.numpy(), g.numpy(), cfg.pad))
    assert rel <= 1e-5 and mx <= 1e-3
    plan.close()


def test_determinism_and_batch_independence():
    cfg = SMALL["c4"]
    x, g = make_inputs(cfg)
    plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, cfg.batch, cfg.padding)
    plan.filter_transform(g.cuda())
    xd = x.cuda()
    y1 = plan.forward(xd).cpu()
    y2 = plan.forward(xd).cpu()
    assert torch.equal(y1, y2)
    y3 = plan.forward(xd[:2].contiguous()).cpu()
    assert torch.equal(y3, y1[:2])
    plan.filter_transform(g.cuda())           # kernel-cache idempotence
    assert torch.equal(plan.forward(xd).cpu(), y1)
    yz = plan.forward(torch.zeros_like(xd)).cpu()
    assert torch.count_nonzero(yz) == 0
    # host-buffer entry point (e2e path) gives the same bits
    yh = torch.empty_like(y1).pin_memory()
    plan.forward_host(x.pin_memory(), yh)
    assert torch.equal(yh, y1)
    plan.close()


def test_error_codes():
    cfg = SMALL["c2"]
    plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, 2, cfg.padding)
    x, g = make_inputs(cfg, batch=2)
    with pytest.raises(pkg.WinoError) as ei:
        plan.forward(x.cuda())
    assert ei.value.status == wino.WINO_ERR_STATE
    plan.filter_transform(g.cuda())
    x3, _ = make_inputs(cfg, batch=3)
    y3 = torch.empty((3, cfg.K) + cfg.out_dims, device="cuda")
    with pytest.raises(pkg.WinoError) as ei:            # the ABI's own check (B > planned batch)
        wino.wino_forward(plan.h, x3.cuda(), y3, 3)
    assert ei.value.status == wino.WINO_ERR_ARG
    # the binding checks every tensor shape before a pointer reaches the ABI
    with pytest.raises(ValueError):
        plan.forward(x3.cuda())                          # batch above the plan's
    with pytest.raises(ValueError):
        plan.forward(x.cuda()[:, :-1].contiguous())      # wrong channel count
    with pytest.raises(ValueError):
        plan.forward(x.cuda(), torch.empty((2, cfg.K + 1) + cfg.out_dims, device="cuda"))   # wrong y
    with pytest.raises(ValueError):
        plan.filter_transform(g.cuda()[:, :, :2].contiguous())                             # wrong g
    with pytest.raises(ValueError):
        plan.forward_host(x, torch.empty((2, cfg.K) + cfg.out_dims[:-1] + (1,)))
    plan.close()


def test_filter_buffer_roundtrip():
    # multi-GPU hook: copying U into a fresh plan + mark_ready == filter_transform
    cfg = SMALL["c3"]
    x, g, y, plan = run(cfg)
    p2 = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, cfg.batch, cfg.padding)
    p2.filter_tensor().copy_(plan.filter_tensor())
    p2.mark_ready()
    assert torch.equal(p2.forward(x.cuda()).cpu(), y)
    plan.close()
    p2.close()


@pytest.mark.parametrize("name", ["c2", "c4", "c5"])
def test_input_cp_async_fallback_matches_tma(name, monkeypatch):
    # the TMA slab load and the cp.async fallback (used when a shape breaks a
    # TMA rule) must produce the same bits
    cfg = SMALL[name]
    x, g, y_tma, plan = run(cfg)
    plan.close()
    monkeypatch.setenv("WINO_IN_TMA", "0")
    _, _, y_cp, plan = run(cfg)
    plan.close()
    assert torch.equal(y_tma, y_cp)


@pytest.mark.parametrize("name", ["c2", "c4", "c5"])
def test_input_slabs_per_cta_bit_identical(name, monkeypatch):
    # a2's slabs per CTA (npl; the last CTA takes the ragged remainder, each
    # slab's TMA box issued by its own lane of warp 0) and its block size only
    # regroup work items: every V element is computed by the same operations,
    # so the output bits must not change
    cfg = SMALL[name]
    y0, info0 = _run_env(cfg, monkeypatch)
    for npl, thr in (("1", "256"), ("3", "320"), ("5", "256"), ("8", "448")):
        y1, info1 = _run_env(cfg, monkeypatch, WINO_IN_NPL=npl, WINO_IN_THREADS=thr)
        assert torch.equal(y0, y1), "npl=%s threads=%s (planned %d)" % (npl, thr, info1["in_planes_per_cta"])


def test_nvtx_range_around_forward(monkeypatch):
    # WINO_NVTX=1: the binding wraps the ABI call in an NVTX range; same result
    cfg = SMALL["c2"]
    y0, _ = _run_env(cfg, monkeypatch)
    y1, _ = _run_env(cfg, monkeypatch, WINO_NVTX="1")
    assert torch.equal(y0, y1)


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_input_line_aligned_items_bit_identical(name, monkeypatch):
    # a2's line-aligned work items (default; item v of a run is tile v - lead,
    # lead = run start mod 32, so every warp stores whole 128-byte lines of V)
    # against the plain item order (WINO_IN_ALIGN=0), also with other slab
    # groupings: only the item -> thread mapping changes, never the arithmetic
    cfg = SMALL[name]
    y0, _ = _run_env(cfg, monkeypatch, WINO_IN_ALIGN="0")
    y1, _ = _run_env(cfg, monkeypatch, WINO_IN_ALIGN="2")     # 2: every a2 path (1, the default: in-place H mode)
    assert torch.equal(y0, y1)
    for npl, thr in (("1", "256"), ("3", "320"), ("4", "448")):
        y2, _ = _run_env(cfg, monkeypatch, WINO_IN_ALIGN="2", WINO_IN_NPL=npl, WINO_IN_THREADS=thr)
        assert torch.equal(y0, y2), "npl=%s threads=%s" % (npl, thr)


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_output_tma_ring_matches_plain(name, monkeypatch):
    # a4 reading M through the TMA ring (alpha^(N-1) >= 32) and through plain
    # per-thread loads: same arithmetic, same bits; also with the L2-chunked
    # pipeline (M rows relative to the chunk) and with several samples per
    # t-block boundary (ragged T)
    cfg = SMALL[name]
    y_tma, _ = _run_env(cfg, monkeypatch)
    y_ld, _ = _run_env(cfg, monkeypatch, WINO_OUT_TMA="0")
    assert torch.equal(y_tma, y_ld)
    monkeypatch.setenv("WINO_FOLD", "0")
    x, g = make_inputs(cfg)
    monkeypatch.setenv("WINO_CHUNK_MB", "0.05")
    plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, cfg.batch, cfg.padding, fuse=4)
    assert plan.info["chunk_slabs"] > 0
    plan.filter_transform(g.cuda())
    assert torch.equal(plan.forward(x.cuda()).cpu(), y_tma)
    plan.close()


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
@pytest.mark.parametrize("chunk_mb", ["0.05", "1"])
def test_l2_chunked_matches_unchunked(name, chunk_mb, monkeypatch):
    # the L2-chunked pipeline (fuse=4) runs the same per-tile arithmetic over
    # slab ranges with chunk-local V/M rows: identical bits for any chunking
    # (compared with the unfused pipeline: chunked plans do not fold, a5)
    monkeypatch.setenv("WINO_FOLD", "0")
    cfg = SMALL[name]
    x, g, y0, plan = run(cfg)
    plan.close()
    monkeypatch.setenv("WINO_CHUNK_MB", chunk_mb)
    _, _, y1, plan = run(cfg, fuse=wino.WINO_FUSE_L2_CHUNK)
    chunks = plan.info["chunk_slabs"]
    plan.close()
    assert torch.equal(y0, y1), "chunk_slabs=%d" % chunks


def _run_env(cfg, monkeypatch, **env):
    # bit-identity tests of the unfused kernels' variants: no a5 fold unless asked
    env.setdefault("WINO_FOLD", "0")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _, _, y, plan = run(cfg)
    info = plan.info
    plan.close()
    for k in env:
        monkeypatch.delenv(k)
    return y, info


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_gemm_variants_bit_identical(name, monkeypatch):
    # the GEMM variants -- A operand from shared memory (0), from TMEM (1),
    # CTA pairs with cta_group::2 (2), U resident or streamed -- issue the same
    # tf32 products in the same order for every output row: identical bits,
    # so the plan's timing-based choice never changes results
    cfg = SMALL[name]
    y_ss, _ = _run_env(cfg, monkeypatch, WINO_GEMM_VARIANT="0")
    y_res, _ = _run_env(cfg, monkeypatch, WINO_GEMM_VARIANT="0", WINO_GEMM_RES="1")
    assert torch.equal(y_ss, y_res)
    y_ts, info = _run_env(cfg, monkeypatch, WINO_GEMM_VARIANT="1")
    assert torch.equal(y_ss, y_ts)
    if info["gemm_variant"] == 1:
        y_tsr, _ = _run_env(cfg, monkeypatch, WINO_GEMM_VARIANT="1", WINO_GEMM_RES="1")
        assert torch.equal(y_ss, y_tsr)
    y_pair, info = _run_env(cfg, monkeypatch, WINO_GEMM_VARIANT="2")
    assert torch.equal(y_ss, y_pair)
    _, info = _run_env(cfg, monkeypatch)
    assert info["gemm_variant"] in (0, 1, 2)


def test_gemm_pair_variant_is_exercised(monkeypatch):
    # c2 / c3 shapes support the CTA-pair kernel (BN = 128): forcing it runs it
    cfg = SMALL["c3"]
    _, info = _run_env(cfg, monkeypatch, WINO_GEMM_VARIANT="2")
    assert info["gemm_variant"] == 2


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
def test_bias_relu_epilogue(name):
    # Eq. (2) with b and f: y = relu(conv + b[k]), fused
    # into the output transform; oracle: direct conv + b, then max(., 0)
    cfg = SMALL[name]
    x, g, y0, plan = run(cfg)
    gen = torch.Generator("cpu").manual_seed(7)
    b = torch.randn(cfg.K, generator=gen, dtype=torch.float32) * 0.1
    xd = x.cuda()
    y_b = plan.forward(xd, bias=b.cuda()).cpu()
    y_br = plan.forward(xd, bias=b.cuda(), relu=True).cpu()
    y_r = plan.forward(xd, relu=True).cpu()
    plan.close()
    ref = direct.direct_conv_f64(x.numpy(), g.numpy(), cfg.pad)
    bb = b.double().numpy().reshape((1, cfg.K) + (1,) * cfg.N)
    tl, tm = tolerance(cfg)
    for y, r in ((y_b, ref + bb), (y_br, np.maximum(ref + bb, 0)), (y_r, np.maximum(ref, 0))):
        rel, mx = errs(y.numpy(), r)
        assert rel <= tl and mx <= tm
    # the epilogue is exact arithmetic on the plain result
    assert torch.equal(y_r, y0.clamp_min(0))
    assert torch.equal(y_b, y0 + b.reshape((1, cfg.K) + (1,) * cfg.N))


def test_gemm_n_tile_choice_bit_identical(monkeypatch):
    # K > 128: the plan also times N tile 128 (where TMEM fits A stages and the
    # CTA-pair kernel applies) against 256; the tile changes which CTA computes
    # an output, never its arithmetic
    from paper_1611_06565_b200.workloads import LayerConfig
    cfg = LayerConfig("k200", 3, 2, 40, 200, (6, 9, 10), 3, 1, 4, "relu_normal", "he")
    y256, info = _run_env(cfg, monkeypatch, WINO_GEMM_VARIANT="0")
    assert info["n_blk"] == 256
    for v in ("0", "1", "2"):
        y128, info = _run_env(cfg, monkeypatch, WINO_GEMM_BN="128", WINO_GEMM_VARIANT=v)
        assert info["n_blk"] == 128
        assert torch.equal(y256, y128)
    y, info = _run_env(cfg, monkeypatch)
    assert torch.equal(y256, y)
    x, g = make_inputs(cfg)
    rel, mx = errs(y.numpy(), direct.direct_conv_f64(x.numpy(), g.numpy(), cfg.pad))
    assert rel <= 1e-5 and mx <= 1e-3


@pytest.mark.parametrize("name,B", [("c1", 1), ("c2", 1), ("c5", 1)])
def test_tiny_single_kernel_path(name, B, monkeypatch):
    # tiny layers can run a2 + a3 + a4 in one kernel (opt-in WINO_TINY=1;
    # fp32 FMA with U_hi + U_lo): within the BJ tolerance of the oracle
    cfg = (CONFIGS if name == "c1" else SMALL)[name]
    x, g = make_inputs(cfg, batch=B)
    ref = direct.direct_conv_f64(x.numpy(), g.numpy(), cfg.pad)
    ys = {}
    for tiny in ("1", "0"):
        monkeypatch.setenv("WINO_TINY", tiny)
        plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, B, cfg.padding)
        ys[tiny] = plan.info["tiny"]
        plan.filter_transform(g.cuda())
        y = plan.forward(x.cuda()).cpu().double().numpy()
        yr = plan.forward(x.cuda(), bias=torch.ones(cfg.K).cuda(), relu=True).cpu().double().numpy()
        plan.close()
        rel = np.linalg.norm(y - ref) / np.linalg.norm(ref)
        tl, tm = tolerance(cfg)
        assert rel <= tl and np.abs(y - ref).max() <= tm * np.abs(ref).max(), (tiny, rel)
        assert np.allclose(yr, np.maximum(y + 1.0, 0.0), rtol=0, atol=1e-6)
    assert ys["0"] == 0
    if name == "c1":
        assert ys["1"] == 1                      # BJ c1 qualifies for the single-kernel path


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_filter_transform_blocked_matches_per_output(name, monkeypatch):
    # a1's blocked kernel (W and the taps staged in shared memory) and the
    # per-output kernel form the same fp64 products in the same order
    cfg = SMALL[name]
    x, g = make_inputs(cfg)
    bufs = []
    for blk in ("1", "0"):
        monkeypatch.setenv("WINO_FILTER_BLK", blk)
        plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, cfg.batch, cfg.padding)
        plan.filter_transform(g.cuda())
        torch.cuda.synchronize()
        bufs.append(plan.filter_tensor().clone().cpu())
        plan.close()
    assert torch.equal(bufs[0], bufs[1])
