import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle, build

    build(ref=False)
    return Oracle("oracle")


@pytest.fixture(scope="session")
def ref():
    from oracle import Oracle

    if not Oracle.available("ref"):
        from oracle import build

        try:
            build(ref=True)
        except Exception:  # pragma: no cover - reference absent on this machine
            pass
    if not Oracle.available("ref"):
        pytest.skip("oracle/_ref/libpbsref.so not built (reference absent here)")
    return Oracle("ref")


GOLDEN = os.path.join(ROOT, "tests", "golden")


# Output tolerances.  bf16 path against the oracle run in fp32
# on the bf16-upcast inputs (unit-Gaussian V); f32 path against the reference's
# own f32 output.  Mean 1e-3 is the survey's bar.  The max stays 2e-2, not the
# survey's 1e-2: the output is stored in bf16, whose half-ulp is 7.8e-3 for
# |o| in [2, 4), and P enters the PV product in bf16; the observed worst case
# over the GPU suite is 1.64e-2 max / 8.5e-4 mean (profiles/r02_output_errors.json).  Every check logs its observed error; with PBS_AUDIT_DIR set
# the log is written to $PBS_AUDIT_DIR/output_errors.json at session end.
BF16_MAX, BF16_MEAN = 2e-2, 1e-3
F32_MAX = 1e-4
ERRLOG = []


def _stats(err):
    if hasattr(err, "detach"):
        err = err.detach().float()
        return float(err.max().item()), float(err.mean().item())
    return float(err.max()), float(err.mean())


def _log(kind, mx, mean, tag):
    ERRLOG.append({"test": os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], "tag": tag,
                   "kind": kind, "max_abs": mx, "mean_abs": mean})


def assert_bf16(err, tag=None, max_abs=None, mean_abs=None):
    mx, mean = _stats(err)
    _log("bf16", mx, mean, tag)
    assert mx <= (max_abs or BF16_MAX) and mean <= (mean_abs or BF16_MEAN), (tag, mx, mean)


def assert_f32(err, tag=None):
    mx, mean = _stats(err)
    _log("f32", mx, mean, tag)
    assert mx <= F32_MAX, (tag, mx, mean)


def pytest_sessionfinish(session, exitstatus):
    out = os.environ.get("PBS_AUDIT_DIR")
    if out and ERRLOG:
        os.makedirs(out, exist_ok=True)
        worst = {k: max((e["max_abs"] for e in ERRLOG if e["kind"] == k), default=None) for k in ("bf16", "f32")}
        worst_mean = {k: max((e["mean_abs"] for e in ERRLOG if e["kind"] == k), default=None)
                      for k in ("bf16", "f32")}
        with open(os.path.join(out, "output_errors.json"), "w") as f:
            json.dump({"bars": {"bf16": [BF16_MAX, BF16_MEAN], "f32": F32_MAX}, "worst_max_abs": worst,
                       "worst_mean_abs": worst_mean, "checks": ERRLOG}, f, indent=1)
