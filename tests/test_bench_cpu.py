"""CPU checks of bench.py's host logic: the roofline numerators come from the
cost model, stage fractions use the right bound and peak, the JSON config
block, and the reference arm's JSON line (the oracle, run on a tiny config)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_1611_06565_b200.workloads import CONFIGS  # noqa: E402

PEAKS = {"hbm_gbs": 6400.0, "bf16": 1600.0, "bf16_sustained": 1500.0, "source": "test"}


def test_stage_bytes_are_the_compulsory_bytes():
    cfg = CONFIGS["c2"]
    sb = bench.stage_bytes(cfg, cfg.batch)
    x, y = 32 * 128 * 56 * 56 * 4, 32 * 128 * 56 * 56 * 4
    V = M = 36 * 128 * (32 * 14 * 14) * 4
    U = 36 * 128 * 128 * 4
    assert sb == {"input_xform": x + V, "gemm": V + U + M, "output_xform": M + y}


def test_roofline_bounds():
    c2, c4 = CONFIGS["c2"], CONFIGS["c4"]
    r = bench.roofline_for(c2, c2.batch, "gemm", 0.05, PEAKS)
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] == 6400.0
    assert r["achieved"] == pytest.approx(bench.stage_bytes(c2, 32)["gemm"] / 0.05e-3 / 1e9, rel=1e-3)
    t = bench.roofline_for(c4, c4.batch, "gemm", 0.4, PEAKS)
    assert t["bound"] == "tensor" and t["unit"] == "TFLOP/s"
    assert t["peak"] == pytest.approx(1600.0 * 1.1 / 2.25 / 3, rel=1e-3)      # 3xTF32 fp32-equivalent
    f = bench.roofline_for(c4, c4.batch, "gemm", 0.3, PEAKS, 4)             # 3xFP16: f16 rate / 3
    assert f["tensor_util"] == pytest.approx(3 * c4.winograd_gemm_flops() / 0.3e-3 / 1e12 / 1600.0, rel=1e-3)
    assert 0 < t["frac"] < 1.5
    o = bench.roofline_for(c4, c4.batch, "output_xform", 0.2, PEAKS)
    assert o["bound"] == "hbm"


def test_cfg_dict_and_parallelism_labels():
    d = bench.cfg_dict(CONFIGS["c2"], 32, 1, "weak")
    assert d["workload"].startswith("c2:") and d["global_batch"] == 32 and d["F"] == "F(4^2,3^2)"
    assert "flushed" in d["l2"]
    s = bench.cfg_dict(CONFIGS["c1"], 1, 4, "strong")
    assert s["parallelism"].startswith("grid 1x4")                    # batch 1 over 4 ranks: K split


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=300,
                         cwd=str(ROOT))
    assert out.returncode == 0, out.stderr
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["metric"] == bench.METRIC and d["unit"] == "TFLOP/s"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["dtype"] == "f64"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself with two ranks
    (torch.distributed.run, 127.0.0.1); both agree on WORLD_SIZE (gloo here)."""
    env = {k: v for k, v in __import__("os").environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"], capture_output=True,
                         text=True, timeout=300, cwd=str(ROOT), env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout                       # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["dry_run"] and d["n_gpus"] == 2
    assert sorted(r["rank"] for r in d["ranks"]) == [0, 1]
    assert all(r["world"] == 2 and r["gpus_arg"] == 2 for r in d["ranks"])


def test_gpus_flag_must_match_world_size():
    env = dict(__import__("os").environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"], capture_output=True,
                         text=True, timeout=300, cwd=str(ROOT), env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


def test_defaults_headline_c4_strong():
    import argparse
    old = sys.argv
    sys.argv = ["bench.py"]
    try:
        a = bench.parse_args()
    finally:
        sys.argv = old
    assert a.config == "c4" and a.scaling == "strong" and a.gpus == 1
    assert set(a.extra.split(",")) == {"c1", "c2", "c3", "c5"}


def test_tensor_util_and_tf32_peak():
    c4 = CONFIGS["c4"]
    pk = dict(PEAKS, tf32_measured=900.0)
    assert bench.tf32_peak(pk) == 900.0                                 # measured above nominal: used
    assert bench.tf32_peak(dict(PEAKS, tf32_measured=100.0)) == pytest.approx(1600.0 * 1.1 / 2.25)
    u = bench.gemm_tensor_util(c4, c4.batch, 0.4, pk)
    assert u == pytest.approx(3 * c4.winograd_gemm_flops() / 0.4e-3 / 1e12 / 900.0)
    r = bench.roofline_for(CONFIGS["c2"], 32, "gemm", 0.05, pk)
    assert "tensor_util" in r and r["bound"] == "hbm"


@pytest.mark.parametrize("name,world", [("c1", 4), ("c2", 2), ("c4", 8), ("c5", 8)])
def test_strong_shards_cover_the_layer_once(name, world):
    """--scaling strong: the ranks' (sample, kernel) shards tile the config's
    batch x K exactly once, with the inputs the single-GPU run would see."""
    from paper_1611_06565_b200.workloads import make_inputs
    cfg = CONFIGS[name].with_batch(min(CONFIGS[name].batch, 8))
    xf, gf = make_inputs(cfg)
    cover = __import__("torch").zeros(cfg.batch, cfg.K, dtype=__import__("torch").int32)
    for rank in range(world):
        x, g, B, Kl, ksplit = bench.layer_shard(cfg, rank, world, "strong")
        assert x.shape[0] == B and g.shape[0] == Kl and ksplit == (Kl != cfg.K)
        from paper_1611_06565_b200.dist import grid_shard
        b_lo, b_hi, k_lo, k_hi = grid_shard(cfg.batch, cfg.K, rank, world)
        assert (x == xf[b_lo:b_hi]).all() and (g == gf[k_lo:k_hi]).all()
        cover[b_lo:b_hi, k_lo:k_hi] += 1
    assert (cover == 1).all()
    xw, gw, Bw, Kw, ks = bench.layer_shard(cfg, 1, world, "weak")
    assert Bw == cfg.batch and Kw == cfg.K and not ks and (gw == gf).all()
