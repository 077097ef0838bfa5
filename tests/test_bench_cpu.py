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
