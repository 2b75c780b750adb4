"""bench.py's JSON line contract: the keys the driver reads, for both arms.

CPU: the reference arm (`--impl reference`, the compiled reference on the host
cores) on a small sample.  GPU: our arm at a reduced sequence length."""
import json
import os
import subprocess
import sys

import pytest

from oracle import Oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _run(*args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.skipif(not Oracle.available("ref"), reason="reference shim not built")
def test_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-seq", "2048")
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["unit"] == "ms" and d["higher_is_better"] is False
    assert d["value"] > 0 and d["config"]["workload"] == "llama31_8b_attn_128k_pbs"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_our_arm_line():
    d = _run("--steps", "2", "--warmup", "3", "--seq", "16384", "--no-cpu-baseline")
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["dtype"] == "bf16"
    assert d["value"] > 0 and d["ms_per_step"] == d["value"] and d["higher_is_better"] is False
    assert d["config"]["workload"] == "llama31_8b_attn_16k_pbs" and "l2" in d["config"]
    r = d["roofline"]
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s" and 0 < r["frac"] < 1.5 and r["peak"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == "ms" and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["speedup_vs_dense_fa"] > 0 and set(d["stage_ms"]) >= {"estimate", "permute", "select", "attention"}
