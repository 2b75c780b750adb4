"""CPU-side checks of the C-ABI library (no GPU needed, no compute calls).

* libpbs_b200.so loads and exports every symbol include/pbs_cabi.h declares;
* host-side validation mirrors PipelineConfig::validate (pipeline.hpp:39-48)
  and returns the reference's exit codes with single-line E_* messages.
"""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "pbs_cabi.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2510_21270_b200 import _lib
    from paper_2510_21270_b200.build import build

    build()
    return _lib.load()


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"PBS_API\s+[\w\s\*]+?\b(pbs_\w+)\s*\(", text)))


def test_header_declares_every_binding():
    from paper_2510_21270_b200._lib import EXPORTS

    assert declared_symbols() == sorted(EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_version(lib):
    assert b"sm_100a" in lib.pbs_version()


def _shape(hq=4, hkv=2, d=128, n=1024, dtype=1):
    from paper_2510_21270_b200._lib import Shape

    return Shape(dtype, hq, hkv, d, n)


def _cfg(**kw):
    from paper_2510_21270_b200.ops import make_config

    return make_config(**kw)


def test_workspace_size_scales(lib):
    a = lib.pbs_workspace_size(C.byref(_shape(n=1024)), C.byref(_cfg()))
    b = lib.pbs_workspace_size(C.byref(_shape(n=2048)), C.byref(_cfg()))
    assert 0 < a < b


@pytest.mark.parametrize("kw,msg", [
    (dict(block_size=0), "block size"),
    (dict(block_size=128, segment_size=100), "segment size"),
    (dict(tau=1.5), "tau"),
    (dict(segment_size=0, strategy="key_permute"), "strategy none"),
    (dict(scale=-1.0), "scale"),
])
def test_config_validation_codes(lib, kw, msg):
    assert lib.pbs_workspace_size(C.byref(_shape()), C.byref(_cfg(**kw))) == 0
    err = lib.pbs_last_error().decode()
    assert err.startswith("E_CONFIG:") and msg in err and "\n" not in err


def test_shape_validation(lib):
    assert lib.pbs_workspace_size(C.byref(_shape(hq=3, hkv=2)), C.byref(_cfg())) == 0
    assert lib.pbs_last_error().decode().startswith("E_SHAPE:")
    rc = lib.pbs_attention(None, None, None, C.byref(_shape(n=0)), C.byref(_cfg()), None, None, None, None, None,
                           0, None, None)
    assert rc == 2


def test_workspace_too_small_is_resource_error(lib):
    rc = lib.pbs_attention(None, None, None, C.byref(_shape()), C.byref(_cfg()), None, None, None, None, None, 16,
                           None, None)
    assert rc == 4 and lib.pbs_last_error().decode().startswith("E_RESOURCE:")


def test_product_has_no_oracle_dependency():
    """The shipped package never imports or links the checker."""
    pkg = os.path.join(ROOT, "paper_2510_21270_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "pbs_oracle" not in text and "libpbsref" not in text, f


def test_cpp_dropin_compiles_and_links(lib, tmp_path):
    """A C++ caller of include/pbs_b200.hpp (the reference-facing wrapper)
    compiles and links against libpbs_b200.so; without a GPU it must fail
    loudly with a single-line E_* error, never fall back to the CPU."""
    import subprocess

    exe = tmp_path / "cpp_dropin"
    pkg = os.path.join(ROOT, "paper_2510_21270_b200")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", "cpp_dropin.cpp"), "-L", pkg, "-lpbs_b200",
           f"-Wl,-rpath,{pkg}", "-o", str(exe)]
    subprocess.run(cmd, check=True)
    import torch

    if not torch.cuda.is_available():
        r = subprocess.run([str(exe), "256", "64"], capture_output=True, text=True)
        assert r.returncode == 1 and r.stderr.startswith("E_CUDA:") and r.stderr.count("\n") == 1


def test_ops_refuse_mismatched_inputs():
    """ops.make_shape: K/V must match Q's N and d (the ABI carries one of each),
    with the reference's error texts (pipeline.hpp:111-116)."""
    import torch

    from paper_2510_21270_b200 import _lib, ops

    q = torch.zeros(4, 256, 64, dtype=torch.bfloat16)
    k = torch.zeros(2, 256, 64, dtype=torch.bfloat16)
    assert ops.make_shape(q, k, k).seq_len == 256
    with pytest.raises(_lib.ConfigError, match="E_CONFIG: pipeline expects self-attention: N == M, got 256 vs 128"):
        ops.make_shape(q, torch.zeros(2, 128, 64, dtype=torch.bfloat16))
    with pytest.raises(_lib.ConfigError, match="E_SHAPE: pipeline inputs have inconsistent shapes"):
        ops.make_shape(q, torch.zeros(2, 256, 32, dtype=torch.bfloat16))
    with pytest.raises(_lib.ConfigError, match="E_SHAPE: pipeline inputs have inconsistent shapes"):
        ops.make_shape(q, k, torch.zeros(2, 200, 64, dtype=torch.bfloat16))
    with pytest.raises(_lib.ConfigError, match="E_SHAPE: num_q_heads"):
        ops.make_shape(q, torch.zeros(3, 256, 64, dtype=torch.bfloat16))
    with pytest.raises(_lib.ConfigError, match="E_CONFIG: Q, K and V must share one dtype"):
        ops.make_shape(q, k.float())
