#!/usr/bin/env python
"""bench.py -- N-D Winograd conv layer F(m^N, r^N) on B200 (arXiv 1611.06565).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c4] [--extra c2,c3,c5,c1] [--scaling strong|weak]

Metric (BASELINE.json): direct-convolution-equivalent TFLOP/s and ms per layer.
A step is one full forward of the layer (stages a2 input transform -> a3
per-point GEMM -> a4 output transform) over one batch that is already
resident in HBM; the filter transform a1 runs once per weight set (the
paper caches transformed kernels) and is reported separately.
The headline workload is c4 (BASELINE.json configs[3], the largest
single-GPU config by direct-equivalent work: the paper's 6x6x6 C3D example,
PAPER.md:191-219); c1, c2, c3 and c5 are reported under "configs".  L2 is
flushed between timed steps, outside the per-step CUDA events: a 256 MiB
memset followed by a 256 MiB read, so the dirty lines of the memset are
written back before the step starts (cold, clean L2;
WINO_BENCH_DIRTY_FLUSH=1 keeps the memset only).

Multi-GPU: one process per GPU over NCCL.  `--gpus N` without a torchrun
environment re-launches this script under `torch.distributed.run` with N
ranks (127.0.0.1 rendezvous).  The batch shards with no per-forward
collective; rank 0 transforms the filters and broadcasts U once (SURVEY.md
8(e)).  "strong" (default): the config batch is split over the ranks (a
(batch x K) grid when the batch is smaller than N); "weak": every rank
convolves a full config-size batch (also reported for the headline config
when N > 1).  Time = max over ranks of device-event time.

--impl reference times the CPU float64 oracle (oracle/, the only reference
that exists for this paper) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from dataclasses import replace
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "direct-equiv TFLOP/s and ms per N-D Winograd conv layer at 1/2/4/8 B200"
GUIDE_TF32_OVER_BF16 = 1.1 / 2.25          # B200_PROFILING.md nominal dense ratio
PARITY_SAMPLES = 4096                       # random outputs per config in the bench's parity block


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--extra", default="c2,c3,c5,c1", help="comma list of further configs ('' for none)")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"])
    ap.add_argument("--dry-run", action="store_true",
                    help="start the ranks, agree on the world size, print one JSON line, exit (no GPU work)")
    ap.add_argument("--no-tf32-peak", action="store_true", help="skip the on-box cuBLAS TF32 peak measurement")
    ap.add_argument("--fuse", type=int, default=0, help="plan fuse bitmask (4 = L2-chunked a2->a3->a4)")
    ap.add_argument("--nets", default="fig4_f54,fig4_f34,fig3_f54",
                    help="the paper's own 2-D workloads (Figures 3 and 4) to time at N=1 ('' for none)")
    ap.add_argument("--nd", default="c3t,c3s133,c3t311",
                    help="per-axis F(m_1 x .. , r_1 x ..) workloads to time at N=1 ('' for none)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the oracle sample")
    return ap.parse_args()


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16": d["bf16_tflops"],
                "bf16_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16": 1590.0, "bf16_sustained": 1400.0, "source": "fallback"}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if self.proc is None:
            return out
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                try:
                    rows.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[3:7]))
                except ValueError:
                    pass
        os.unlink(self.path)
        if not rows:
            return out
        busy = [r for r in rows if r[2] >= 30.0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in busy for i, v in enumerate(r[3]) if v.lower().startswith("active")})
        out.update(sm_mhz=statistics.median(r[0] for r in busy), sm_max_mhz=max(r[1] for r in rows),
                   reasons=reasons, samples=len(busy))
        return out


# ------------------------------------------------------------------ helpers
def stage_model_for(cfg, B, info=None):
    """The package's analytic cost model of the plan as built (DESIGN.md
    Sec. 8): with an a5 fold (info "fold" / "fold_mode") the GEMM writes and
    a4 reads W instead of M, and the filter-side fold streams U' and executes
    m^F x the multiply-adds."""
    from paper_1611_06565_b200.cost import stage_model
    info = info or {}
    return stage_model(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, B, cfg.padding,
                       fold=info.get("fold", 0), fold_mode=info.get("fold_mode", 0))


def stage_bytes(cfg, B, info=None):
    """Algorithmic (compulsory) bytes of each stage for B samples."""
    st = stage_model_for(cfg, B, info)
    return {s: st[s]["bytes"] for s in ("input_xform", "gemm", "output_xform")}


def tf32_peak(peaks):
    """TF32 dense peak (TFLOP/s) for the per-point GEMM's roofline: the larger
    (more conservative) of the on-box cuBLAS TF32 measurement and the measured
    bf16 peak x the guide's nominal TF32/bf16 ratio."""
    nominal = peaks["bf16"] * GUIDE_TF32_OVER_BF16
    return max(nominal, peaks.get("tf32_measured") or 0.0)


WINO_GEMM_3XF16 = 4


def gemm_pipe_peak(peaks, gemm_mode=3):
    """Dense peak (TFLOP/s) of the tensor kind the GEMM scheme runs on: TF32
    for 3xTF32, the measured bf16 peak (= f16 dense rate) for 3xFP16."""
    return peaks["bf16"] if gemm_mode == WINO_GEMM_3XF16 else tf32_peak(peaks)


def gemm_tensor_util(cfg, B, ms, peaks, gemm_mode=3, info=None):
    """Tensor-pipe utilisation of the per-point GEMM: 3 tensor products per
    fp32 multiply-add (3xTF32 or 3xFP16), 3 * 2 alpha^N T C K / (t * peak of
    that tensor kind); the multiply-adds the GEMM executes (m^F x under the
    filter-side fold)."""
    flops = stage_model_for(cfg, B, info)["gemm"]["flops"]
    return 3 * flops / (ms * 1e-3) / 1e12 / gemm_pipe_peak(peaks, gemm_mode)


def roofline_for(cfg, B, stage, ms, peaks, gemm_mode=3, info=None):
    t = ms * 1e-3
    sm = stage_model_for(cfg, B, info)
    nbytes = sm[stage]["bytes"]
    tf32 = gemm_pipe_peak(peaks, gemm_mode)
    if stage == "gemm":
        flops = sm["gemm"]["flops"]
        t_mem = nbytes / (peaks["hbm_gbs"] * 1e9)
        t_tc = flops / (tf32 / 3 * 1e12)
        util = round(gemm_tensor_util(cfg, B, ms, peaks, gemm_mode, info), 4)
        if t_tc > t_mem:
            ach = flops / t / 1e12
            return {"bound": "tensor", "achieved": round(ach, 2), "peak": round(tf32 / 3, 1), "unit": "TFLOP/s",
                    "frac": round(ach / (tf32 / 3), 4), "traffic": None, "tensor_util": util,
                    "note": ("fp32 flops of the per-point GEMM vs the 3xFP16 fp32-equivalent peak = f16 (= bf16 %s) "
                             "dense peak / 3" % peaks["source"]) if gemm_mode == WINO_GEMM_3XF16 else
                            ("fp32 flops of the per-point GEMM vs the 3xTF32 fp32-equivalent peak = TF32 peak / 3; "
                             "TF32 peak = max(on-box cuBLAS TF32, bf16 %s x 1.1/2.25)" % peaks["source"])}
        ach = nbytes / t / 1e9
        return {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(ach / peaks["hbm_gbs"], 4), "traffic": None, "tensor_util": util}
    ach = nbytes / t / 1e9
    return {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": round(ach / peaks["hbm_gbs"], 4), "traffic": None}


def measure_tf32_peak(dev):
    """cuBLAS fp32 matmul with TF32 tensor cores, 8192^3, best of 10 (CUDA
    events): the on-box TF32 dense peak."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        n = 8192
        a = torch.randn(n, n, device=dev)
        b = torch.randn(n, n, device=dev)
        c = torch.empty(n, n, device=dev)
        for _ in range(3):
            torch.matmul(a, b, out=c)
        best = 1e30
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b, out=c)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b, c
        torch.cuda.empty_cache()
        return 2 * n ** 3 / (best * 1e-3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def load_traffic():
    p = ROOT / "profiles" / "ncu_traffic.json"
    return json.loads(p.read_text()) if p.exists() else {}


# ------------------------------------------------------------------ ours
def layer_shard(cfg, rank, world, scaling):
    """This rank's inputs: (x, g, B, K_local, ksplit).
    weak: a full config batch per rank (x seeded by rank, the same g);
    strong: the config batch over the ranks, and when the batch is smaller
    than the world the output channels too (dist.grid_shard, NEXT-3)."""
    from paper_1611_06565_b200 import dist as wdist
    from paper_1611_06565_b200.workloads import make_inputs
    if scaling == "weak":
        x = make_inputs(cfg, seed=rank)[0]
        g = make_inputs(cfg, seed=0)[1]              # same weights on every rank
        return x, g, cfg.batch, cfg.K, False
    b_lo, b_hi, k_lo, k_hi = wdist.grid_shard(cfg.batch, cfg.K, rank, world)
    xf, gf = make_inputs(cfg, seed=0)
    return (xf[b_lo:b_hi].contiguous(), gf[k_lo:k_hi].contiguous(), b_hi - b_lo, k_hi - k_lo,
            k_hi - k_lo != cfg.K)


def run_ours(args, cfg_names, rank, world, local, peaks, scaling=None):
    import torch
    import paper_1611_06565_b200 as pkg
    from paper_1611_06565_b200 import dist as wdist
    from paper_1611_06565_b200.workloads import CONFIGS, make_inputs

    dev = torch.device("cuda", local)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush64 = flush.view(torch.int64)
    flush_sink = torch.empty((), dtype=torch.int64, device=dev)
    clean = os.environ.get("WINO_BENCH_DIRTY_FLUSH", "0") != "1"

    def l2_flush():
        # write 256 MiB (> 126 MB L2), then read it back: the read evicts (and
        # writes back) the dirty lines of the write, so every step starts with
        # a cold *and clean* L2 -- the state ncu's --cache-control all gives
        flush.zero_()
        if clean:
            torch.sum(flush64, dim=0, out=flush_sink)

    scaling = scaling or args.scaling
    results = {}
    for name in cfg_names:
        cfg = CONFIGS[name]
        x, g, B, Kl, ksplit = layer_shard(cfg, rank, world, scaling)
        plan = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, Kl, B, cfg.padding, device=local, fuse=args.fuse)
        stream = torch.cuda.current_stream(dev)
        # a1 once per weight set on rank 0, U broadcast over NCCL to the
        # others; with a K split every rank transforms its own kernel slice
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if rank == 0 or ksplit:
            gd = g.to(dev)
            plan.filter_transform(gd, stream)          # first call (module load), then timed
            e0.record(stream)
            plan.filter_transform(gd, stream)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            filt_ms = e0.elapsed_time(e1)
        else:
            filt_ms = None
        if not ksplit:
            wdist.broadcast_filter(plan.filter_tensor(), src=0)
        torch.cuda.synchronize(dev)
        if rank != 0 and not ksplit:
            plan.mark_ready()
        xd = x.to(dev)
        y = torch.empty((B, Kl) + cfg.out_dims, device=dev, dtype=torch.float32)
        for _ in range(max(args.warmup, 3)):
            plan.forward(xd, y, stream)
        torch.cuda.synchronize(dev)
        # ---- timed region: K steps, barrier + sync on both sides.  No events
        # between the kernels of a step (they would break the programmatic
        # dependent launches); per-stage times come from a separate pass.
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        wdist.barrier(device=dev)
        torch.cuda.synchronize(dev)
        for i in range(args.steps):
            l2_flush()                                 # L2 flush, outside the step events
            evs[i][0].record(stream)
            plan.forward(xd, y, stream)
            evs[i][1].record(stream)
        torch.cuda.synchronize(dev)
        wdist.barrier(device=dev)
        step_ms = [a.elapsed_time(b) for a, b in evs]
        # ---- instrumented pass: CUDA events around every stage launch
        plan.profile(True)
        for i in range(max(3, min(args.steps, 10))):
            l2_flush()
            plan.forward(xd, y, stream)
        torch.cuda.synchronize(dev)
        stage_ms, calls = plan.profile_read()
        plan.profile(False)
        ms_local = sum(step_ms) / len(step_ms)
        ms = wdist.max_over_ranks(ms_local, device=dev)
        stages = dict(zip(["input_xform", "gemm", "output_xform"], [s / calls for s in stage_ms]))
        # ---- end to end through the public C ABI with host buffers
        xh = x.pin_memory()
        yh = torch.empty((B, Kl) + cfg.out_dims, dtype=torch.float32).pin_memory()
        for _ in range(2):
            plan.forward_host(xh, yh, stream)
        wdist.barrier(device=dev)
        ee = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(max(3, min(args.steps, 20)))]
        for a, b in ee:
            a.record(stream)
            plan.forward_host(xh, yh, stream)
            b.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms = wdist.max_over_ranks(sum(a.elapsed_time(b) for a, b in ee) / len(ee), device=dev)
        # whole-job flops: weak = world x one config batch; strong = one config batch
        flops_job = world * cfg.direct_flops(B) if scaling == "weak" else cfg.direct_flops()
        # outputs of the last forward at sampled positions (every output for
        # small layers), for the parity block computed by the cpu_baseline leg
        sample = None
        if world == 1:
            yf = yh.view(-1)
            n_out = yf.numel()
            if n_out <= (1 << 16):
                idx = torch.arange(n_out)
            else:
                gen = torch.Generator("cpu").manual_seed(1)
                idx = torch.cat([torch.arange(64), torch.arange(n_out - 64, n_out),
                                 torch.randint(0, n_out, (PARITY_SAMPLES,), generator=gen)])
            sample = (idx.numpy(), yf[idx].double().numpy())
        res = {
            "name": name, "cfg": cfg, "cfg_local": replace(cfg, K=Kl), "B": B, "ms": ms, "tflops": flops_job / (ms * 1e-3) / 1e12, "K_local": Kl,
            "stages_ms": stages, "filter_ms": filt_ms, "e2e_ms": e2e_ms,
            "e2e_tflops": flops_job / (e2e_ms * 1e-3) / 1e12,
            "h2d": xh.numel() * 4, "d2h": yh.numel() * 4, "launches": plan.launches_per_forward * args.steps,
            "sample": sample, "scaling": scaling,
            "info": plan.info,
        }
        results[name] = res
        plan.close()
        del xd, y
        torch.cuda.empty_cache()
    return results


# Figure 4 of the paper: 10.9 MVox/s on 18 cores of a Xeon E7-8890, context only
PAPER_FIG4_MVOX = 10.9


def run_nets(args, local):
    """The paper's own 2-D workloads (workloads.NETS): each net at each of its
    batch sizes, device-resident, L2 flushed before every pass, CUDA events
    around the whole chain of layers.  MVox/s = batch x input voxels / time
    (reading #16)."""
    import torch
    import paper_1611_06565_b200 as pkg
    from paper_1611_06565_b200.workloads import NETS, make_net_inputs
    dev = torch.device("cuda", local)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    sink = torch.empty((), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    steps = max(3, min(args.steps, 20))
    out = {}
    for name in [n for n in args.nets.split(",") if n]:
        net_cfg = NETS[name]
        rows = {}
        for B in net_cfg.batches:
            x, gs = make_net_inputs(net_cfg, seed=0, batch=B)
            layers = [(l.N, l.dims, l.m, l.r, l.C, l.K, l.padding) for l in net_cfg.layers]
            net = pkg.Net(layers, B, device=local)
            net.filter_transform([g.to(dev) for g in gs], stream)
            xd = x.to(dev)
            for _ in range(max(args.warmup, 3)):
                net.forward(xd, stream)
            torch.cuda.synchronize(dev)
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            for a, b in evs:
                flush.zero_()
                torch.sum(flush.view(torch.int64), dim=0, out=sink)
                a.record(stream)
                net.forward(xd, stream)
                b.record(stream)
            torch.cuda.synchronize(dev)
            ms = sum(a.elapsed_time(b) for a, b in evs) / steps
            # the same pass replayed from a CUDA graph (Net.capture)
            replay = net.capture(xd)
            for _ in range(3):
                replay()
            torch.cuda.synchronize(dev)
            for a, b in evs:
                flush.zero_()
                torch.sum(flush.view(torch.int64), dim=0, out=sink)
                a.record(stream)
                replay()
                b.record(stream)
            torch.cuda.synchronize(dev)
            ms_g = sum(a.elapsed_time(b) for a, b in evs) / steps
            best = min(ms, ms_g)
            rows[str(B)] = {"ms_per_pass": round(ms, 4), "ms_per_pass_graph": round(ms_g, 4),
                            "mvox_s": round(B * net_cfg.in_voxels / (best * 1e-3) / 1e6, 1),
                            "tflops_direct_equiv": round(net_cfg.direct_flops(B) / (best * 1e-3) / 1e12, 2),
                            "gemm_variants": [p.info["gemm_variant"] for p in net.plans]}
            del replay
            net.close()
            del xd
            torch.cuda.empty_cache()
        best = max(rows.values(), key=lambda r: r["mvox_s"])
        out[name] = {"desc": net_cfg.desc, "layers": len(net_cfg.layers),
                     "F": "F(%d^2,%d^2)" % (net_cfg.layers[0].m, net_cfg.layers[0].r),
                     "by_batch": rows, "best_mvox_s": best["mvox_s"]}
        if name.startswith("fig4"):
            out[name]["paper_mvox_s"] = {"value": PAPER_FIG4_MVOX, "hardware": "18-core Xeon E7-8890 (context only)"}
    return out


# Per-axis workloads (NEXT-2): c3's video layer with F(2,3) along time and
# F(4,3) along space (Eq. (4)'s per-axis transforms)
ND_WORKLOADS = {
    "c3t": dict(N=3, dims=(16, 56, 56), m=(2, 4, 4), r=(3, 3, 3), pad=(1, 1, 1), B=16, C=64, K=128,
                desc="c3 video layer 16x56x56, 16x64->128, F(2,3) time x F(4x4,3x3) space"),
    # the (2+1)-D factorisation of the same layer: a 1x3x3 spatial and a
    # 3x1x1 temporal convolution (anisotropic kernels; F(1,1) is the identity)
    "c3s133": dict(N=3, dims=(16, 56, 56), m=(1, 4, 4), r=(1, 3, 3), pad=(0, 1, 1), B=16, C=64, K=128,
                   desc="1x3x3 spatial kernel on c3's input, 16x64->128, F(1,1) x F(4x4,3x3)"),
    "c3t311": dict(N=3, dims=(16, 56, 56), m=(4, 1, 1), r=(3, 1, 1), pad=(1, 0, 0), B=16, C=64, K=128,
                   desc="3x1x1 temporal kernel on c3's input, 16x64->128, F(4,3) x F(1,1)^2"),
}


def run_nd(args, local, peaks=None):
    import torch
    import paper_1611_06565_b200 as pkg
    dev = torch.device("cuda", local)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    sink = torch.empty((), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    steps = max(3, min(args.steps, 20))
    out = {}
    for name in [n for n in args.nd.split(",") if n]:
        w = ND_WORKLOADS[name]
        gen = torch.Generator("cpu").manual_seed(0)
        x = torch.randn((w["B"], w["C"]) + w["dims"], generator=gen)
        g = torch.randn((w["K"], w["C"]) + w["r"], generator=gen) * math.sqrt(2.0 / (w["C"] * math.prod(w["r"])))
        plan = pkg.Plan(w["N"], w["dims"], list(w["m"]), list(w["r"]), w["C"], w["K"], w["B"], w["pad"],
                        device=local)
        plan.filter_transform(g.to(dev), stream)
        xd = x.to(dev)
        y = torch.empty((w["B"], w["K"]) + tuple(plan.out_dims), device=dev)
        for _ in range(max(args.warmup, 3)):
            plan.forward(xd, y, stream)
        torch.cuda.synchronize(dev)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a, b in evs:
            flush.zero_()
            torch.sum(flush.view(torch.int64), dim=0, out=sink)
            a.record(stream)
            plan.forward(xd, y, stream)
            b.record(stream)
        torch.cuda.synchronize(dev)
        ms = sum(a.elapsed_time(b) for a, b in evs) / steps
        plan.profile(True)
        for _ in range(3):
            plan.forward(xd, y, stream)
        torch.cuda.synchronize(dev)
        stage_ms, calls = plan.profile_read()
        plan.profile(False)
        flops = 2 * w["B"] * w["K"] * w["C"] * math.prod(plan.out_dims) * math.prod(w["r"])
        # per-stage roofline fractions from the cost model's compulsory bytes / flops
        from paper_1611_06565_b200.cost import stage_model
        pk = peaks or load_peaks()
        tf32 = tf32_peak(pk)
        sm = stage_model(w["N"], w["dims"], w["m"], w["r"], w["C"], w["K"], w["B"], w["pad"],
                         hbm_gbs=pk["hbm_gbs"], tf32_tflops=tf32)
        frac = {}
        for sname, v in zip(["input_xform", "gemm", "output_xform"], stage_ms):
            t_ms = v / calls
            frac[sname] = round(sm[sname]["roofline_ms"] / t_ms, 3) if t_ms > 0 else None
        out[name] = {"desc": w["desc"], "F": "F(%s, %s)" % ("x".join(map(str, w["m"])), "x".join(map(str, w["r"]))),
                     "ms_per_layer": round(ms, 4), "tflops_direct_equiv": round(flops / (ms * 1e-3) / 1e12, 2),
                     "n_points": plan.info["n_points"],
                     "stages_ms": {s: round(v / calls, 4) for s, v in
                                   zip(["input_xform", "gemm", "output_xform"], stage_ms)},
                     "stages_roofline_frac": frac,
                     "path": {0: "single F(m, r) fused kernels",
                              1: "fused kernels with a distinct axis-0 transform (xform_mixed.cu)",
                              2: "generic multi-pass per-axis transforms (xform_nd.cu)"}[plan.info["axis_mode"]]
                             + " + tcgen05 3xTF32 GEMM"}
        plan.close()
        del xd, y
        torch.cuda.empty_cache()
    return out


def cpu_baseline_leg(results, head, seconds):
    """The cpu_baseline leg: the float64 oracle (as it stands, OpenMP on the
    host cores) evaluated one output at a time at the positions bench.py kept
    from each config's last end-to-end forward.  Its timing on the headline
    config (extended to a bounded sample of about `seconds` of CPU work) is
    the reported CPU baseline; the same oracle values give the parity block
    (relL2 and max-abs / max|y| over the sampled outputs, in float64;
    full-size element-wise checks are in tests/test_gpu_parity.py)."""
    import numpy as np
    from oracle import direct
    from paper_1611_06565_b200.workloads import make_inputs, tolerance
    parity = {}
    cpu = None
    for name, r in results.items():
        if r.get("sample") is None:
            continue
        cfg = r["cfg"]
        x, g = make_inputs(cfg)
        xn, gn = x.numpy(), g.numpy()
        idx, y_gpu = r["sample"]
        t0 = time.perf_counter()
        ref = direct.direct_conv_at(xn, gn, cfg.pad, idx)
        dt = time.perf_counter() - t0
        err = y_gpu - ref
        rel = float(np.linalg.norm(err) / np.linalg.norm(ref))
        mx = float(np.abs(err).max() / np.abs(ref).max())
        tl, tm = tolerance(cfg)
        n_out = cfg.batch * cfg.K * math.prod(cfg.out_dims)
        parity[name] = {"F": "F(%d^%d,%d^%d)" % (cfg.m, cfg.N, cfg.r, cfg.N), "relL2": float("%.3e" % rel),
                        "max_over_maxy": float("%.3e" % mx), "tol": [tl, tm], "pass": rel <= tl and mx <= tm,
                        "outputs": "all %d" % n_out if len(idx) == n_out else
                                   "%d sampled of %d (first/last 64 + random)" % (len(idx), n_out)}
        if name == head:
            per_pt = 2 * cfg.C * cfg.r ** cfg.N
            npts = len(idx)
            if dt < seconds * 0.5:          # extend to a bounded sample of ~`seconds` of CPU work
                rng = np.random.default_rng(0)
                npts = int(min(n_out, max(len(idx), len(idx) * (seconds * 0.8) / max(dt, 1e-3))))
                more = rng.integers(0, n_out, npts)
                t0 = time.perf_counter()
                direct.direct_conv_at(xn, gn, cfg.pad, more)
                dt = time.perf_counter() - t0
            cpu = {"value": round(npts * per_pt / dt / 1e12, 6), "unit": "TFLOP/s", "cores": direct.num_threads(),
                   "cpu_model": cpu_model(), "kind": "oracle", "seconds": round(dt, 2),
                   "sample": "%d random outputs of %s (of %d), float64 direct correlation, OpenMP"
                             % (npts, cfg.name, n_out),
                   "ms_per_layer_extrapolated": round(cfg.direct_flops() / (npts * per_pt / dt) * 1e3, 1)}
    return cpu, parity


def cfg_dict(cfg, B, world, scaling, fuse=0):
    from paper_1611_06565_b200.dist import grid_shape
    if scaling == "weak" or cfg.batch >= world:
        par = "dp%d (batch shards, U broadcast once)" % world
    else:
        par = "grid %dx%d (batch shards x output-channel shards, no reduction)" % grid_shape(cfg.batch, cfg.K, world)
    return {"workload": "%s: %s" % (cfg.name, cfg.desc), "model": "N-D Winograd conv layer (synthetic)",
            "N": cfg.N, "dims": list(cfg.dims), "C": cfg.C, "K": cfg.K, "kernel": cfg.r, "pad": cfg.pad,
            "F": "F(%d^%d,%d^%d)" % (cfg.m, cfg.N, cfg.r, cfg.N), "per_gpu_batch": B,
            "global_batch": B * world if scaling == "weak" else cfg.batch, "seq_len": None,
            "parallelism": par,
            "gemm": "tcgen05, TMEM fp32 accumulation; scheme per config (configs.*.gemm_scheme): 3xTF32 (variant "
                    "timed at plan creation: 0 SMEM-A, 1 TMEM-A, 2 CTA-pair) or 3xFP16 (power-of-two scaled fp16 "
                    "hi/lo split on kind::f16, CTA pairs) where measured faster; F(2^N,3^N), N >= 3: output "
                    "transform of the 2 innermost axes in the GEMM epilogue (a5)",
            "pipeline": "L2-chunked a2->a3->a4" if fuse & 4 else "three kernels, V/M via HBM",
            "l2": ("flushed: 256 MiB memset + 256 MiB read (cold, clean L2) between timed steps, "
                   "outside the per-step events") if os.environ.get("WINO_BENCH_DIRTY_FLUSH", "0") != "1"
                  else "flushed: 256 MiB memset between timed steps, outside the per-step events"}


def free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def relaunch_under_torchrun(n):
    """`--gpus N` without a torchrun environment: re-run this script with N
    ranks, one per GPU, under torch.distributed.run (127.0.0.1 rendezvous)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), str(Path(__file__).resolve())]
    cmd += sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "8")
    return subprocess.call(cmd, env=env)


def dry_run(args, rank, world, local):
    """Start the process group, agree on the world size, print one line."""
    import torch
    import torch.distributed as dist
    use_nccl = torch.cuda.is_available() and torch.cuda.device_count() > local
    if world > 1:
        if use_nccl:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
        got = [None] * world
        dist.all_gather_object(got, {"rank": rank, "world": world, "gpus_arg": args.gpus})
        dist.destroy_process_group()
    else:
        got = [{"rank": 0, "world": 1, "gpus_arg": args.gpus}]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "backend": ("nccl" if use_nccl else "gloo")
                          if world > 1 else None, "ranks": got}))
    return 0


def main():
    args = parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch_under_torchrun(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE=%d (launch with --nproc-per-node %d, or drop "
                         "the torchrun environment)" % (args.gpus, world, args.gpus))
    from paper_1611_06565_b200.workloads import CONFIGS

    if args.impl == "reference":
        if rank != 0:
            return 0
        return run_reference(args, world)
    if args.dry_run:
        return dry_run(args, rank, world, local)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL's INIT log (to stderr: stdout carries the JSON line) shows the
        # communicator's nranks / transport
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks = load_peaks()
    if not args.no_tf32_peak:
        tf = measure_tf32_peak(torch.device("cuda", local))
        peaks["tf32_measured"] = wdist_max(tf, world, local)
    names = [args.config] + [n for n in args.extra.split(",") if n and n != args.config]
    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    res = run_ours(args, names, rank, world, local, peaks)
    clocks = sampler.stop() if rank == 0 else None
    weak = None
    if world > 1 and args.scaling == "strong":
        weak = run_ours(args, [args.config], rank, world, local, peaks, scaling="weak")[args.config]
    if world > 1:
        dist.barrier()
    if rank == 0:
        traffic = load_traffic()
        head = res[args.config]
        cfg = head["cfg"]
        out = {"metric": METRIC, "value": round(head["tflops"], 3), "unit": "TFLOP/s", "n_gpus": world,
               "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(head["ms"], 5),
               "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
               "data": "synthetic (seeded, BASELINE.json distributions; no dataset)",
               "config": cfg_dict(cfg, head["B"], world, args.scaling, args.fuse)}
        configs = {}
        for name, r in res.items():
            st = r["stages_ms"]
            dom = max(st, key=st.get)
            gm = r["info"]["gemm_mode"]
            rl = roofline_for(r["cfg_local"], r["B"], dom, st[dom], peaks, gm, r["info"])
            rl["kernel"] = dom
            tk = traffic.get(name, {}).get(dom)
            if tk is not None:
                rl["traffic"] = tk
            # a tiny plan runs the three stages in one kernel (timed as "gemm")
            per_stage = {}
            for sname, v in st.items():
                if v <= 0:
                    per_stage[sname] = {"ms": 0.0, "note": "fused into the single-kernel tiny path"}
                    continue
                rf = roofline_for(r["cfg_local"], r["B"], sname, v, peaks, gm, r["info"])
                per_stage[sname] = {"ms": round(v, 5), **{k: rf[k] for k in ("bound", "achieved", "unit", "frac")}}
                if sname == "gemm":
                    per_stage[sname]["tensor_util"] = rf["tensor_util"]
            configs[name] = {"ms_per_layer": round(r["ms"], 5), "tflops_direct_equiv": round(r["tflops"], 2),
                             "stages": per_stage, "dominant": rl,
                             "filter_transform_ms": None if r["filter_ms"] is None else round(r["filter_ms"], 4),
                             "e2e_tflops": round(r["e2e_tflops"], 3), "e2e_ms": round(r["e2e_ms"], 4),
                             "gemm_scheme": {3: "3xTF32", 4: "3xFP16 (scaled split)", 1: "FFMA"}.get(gm, str(gm)),
                             "info": {k: r["info"][k] for k in ("T_per_sample", "n_points", "n_blk", "k_chunk",
                                                                 "chunk_slabs", "gemm_variant", "in_slab_tiles",
                                                                 "in_planes_per_cta", "axis_mode", "tiny", "fold", "fold_mode", "in_bands")}}
        out["roofline"] = configs[args.config]["dominant"]
        out["roofline"]["peak_source"] = ("HBM: MEASURED_PEAKS.json (%s); tensor: TF32 = max(on-box cuBLAS "
                                          "TF32 %s, bf16 x 1.1/2.25)" % (
                                              peaks["source"], "%.1f TFLOP/s" % peaks["tf32_measured"]
                                              if peaks.get("tf32_measured") else "not measured"))
        if world == 1 and not args.no_cpu_baseline:
            cpu, parity = cpu_baseline_leg(res, args.config, args.cpu_seconds)
            out["cpu_baseline"] = cpu
            out["parity"] = parity
        out["e2e"] = {"value": round(head["e2e_tflops"], 3), "unit": "TFLOP/s",
                      "h2d_bytes_per_step": head["h2d"], "d2h_bytes_per_step": head["d2h"],
                      "ms_per_step": round(head["e2e_ms"], 4),
                      "path": "wino_forward_host (pinned host buffers, H2D + forward + D2H + sync)"}
        out["gpu_launches"] = head["launches"]
        out["clocks"] = clocks
        out["peaks"] = {"hbm_gbs": peaks["hbm_gbs"], "bf16_tflops": peaks["bf16"],
                        "tf32_tflops_measured": None if not peaks.get("tf32_measured")
                        else round(peaks["tf32_measured"], 1),
                        "tf32_tflops_used": round(tf32_peak(peaks), 1)}
        out["filter_transform_ms"] = configs[args.config]["filter_transform_ms"]
        out["stages"] = configs[args.config]["stages"]
        out["configs"] = configs
        if weak is not None:
            out["weak_scaling"] = {"config": args.config, "per_gpu_batch": weak["B"],
                                   "global_batch": weak["B"] * world, "ms_per_layer": round(weak["ms"], 5),
                                   "value": round(weak["tflops"], 3), "unit": "TFLOP/s"}
        if world == 1 and args.nets:
            out["paper_workloads"] = run_nets(args, local)
        if world == 1 and args.nd:
            out["per_axis_workloads"] = run_nd(args, local, peaks)
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()
    return 0


def wdist_max(v, world, local):
    if world == 1:
        return v
    from paper_1611_06565_b200 import dist as wdist
    import torch
    return wdist.max_over_ranks(v, device=torch.device("cuda", local))


def run_reference(args, world):
    """The float64 oracle as the reference arm, each step a bounded sample."""
    import numpy as np
    from oracle import direct
    from paper_1611_06565_b200.workloads import CONFIGS, make_inputs
    cfg = CONFIGS[args.config]
    x, g = make_inputs(cfg)
    xn, gn = x.numpy(), g.numpy()
    per_pt = 2 * cfg.C * cfg.r ** cfg.N
    n_out = cfg.batch * cfg.K * math.prod(cfg.out_dims)
    rng = np.random.default_rng(0)
    npts = max(256, int(1.5e9 / per_pt))          # ~1.5 GFLOP of f64 work per step
    for _ in range(max(args.warmup, 1)):
        direct.direct_conv_at(xn, gn, cfg.pad, rng.integers(0, n_out, min(npts, 4096)))
    times = []
    for _ in range(args.steps):
        idx = rng.integers(0, n_out, npts)
        t0 = time.perf_counter()
        direct.direct_conv_at(xn, gn, cfg.pad, idx)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = npts * per_pt / (ms * 1e-3) / 1e12
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "TFLOP/s", "n_gpus": world,
           "steps": args.steps, "warmup": max(args.warmup, 1), "ms_per_step": round(ms, 3),
           "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded, BASELINE.json distributions; no dataset)",
           "config": cfg_dict(cfg, cfg.batch, 1, args.scaling),
           "cpu_baseline": {"value": round(value, 6), "unit": "TFLOP/s", "cores": direct.num_threads(),
                            "kind": "oracle",
                            "sample": "%d random outputs of %s per step (float64 direct correlation)" % (npts, cfg.name)},
           "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "ms_per_layer_extrapolated": round(cfg.direct_flops() / (value * 1e12) * 1e3, 1)}
    print(json.dumps(out))
    return 0


if __name__ == "__main__":
    sys.exit(main())
