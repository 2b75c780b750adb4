"""PBST tensor files (tensor_io.hpp) through the C ABI, against the reference's
own read_tensor / write_tensor (oracle/_ref, the unmodified headers).

CPU: header parsing and every read_tensor error (code and E_* text, byte
offsets included).  GPU: payloads loaded to / saved from device memory in f32
and bf16, f32 and f64 files, a multi-chunk file, and the non-finite check."""
import ctypes as C
import os
import struct

import numpy as np
import pytest

from oracle import Oracle, OracleError

pytestmark = pytest.mark.skipif(not Oracle.available("ref"), reason="reference shim not built")


@pytest.fixture(scope="module")
def ref():
    return Oracle("ref")


@pytest.fixture(scope="module")
def lib():
    from paper_2510_21270_b200 import _lib
    return _lib.load()


def header(dtype=0, dims=(2, 3, 4), version=1, magic=b"PBST"):
    return magic + struct.pack("<III", version, dtype, len(dims)) + b"".join(struct.pack("<Q", x) for x in dims)


def info(lib, path):
    from paper_2510_21270_b200 import _lib
    i = _lib.TensorInfo()
    rc = lib.pbs_tensor_info_read(str(path).encode(), C.byref(i))
    return rc, (lib.pbs_last_error().decode() if rc else i.as_dict())


def test_header_of_reference_files(ref, lib, tmp_path):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((3, 5, 7)).astype(np.float32)
    ref.write_tensor(tmp_path / "s.pbst", a)
    rc, i = info(lib, tmp_path / "s.pbst")
    assert rc == 0 and i == {"file_dtype": 0, "ndim": 3, "heads": 3, "rows": 5, "cols": 7, "payload_offset": 40}
    b = rng.standard_normal((4, 6))
    ref.write_tensor(tmp_path / "m.pbst", b)
    rc, i = info(lib, tmp_path / "m.pbst")
    assert rc == 0 and i == {"file_dtype": 1, "ndim": 2, "heads": 1, "rows": 4, "cols": 6, "payload_offset": 32}


PAYLOAD = np.zeros(24, dtype=np.float32).tobytes()
MALFORMED = {
    "bad_magic": b"PBSX" + header()[4:] + PAYLOAD,
    "short_magic": b"PB",
    "no_version": b"PBST\x01\x00",
    "bad_version": header(version=2) + PAYLOAD,
    "no_dtype": b"PBST" + struct.pack("<I", 1) + b"\x00\x00",
    "bad_dtype": header(dtype=7) + PAYLOAD,
    "no_ndim": b"PBST" + struct.pack("<II", 1, 0),
    "bad_ndim": header(dims=(1, 2, 3, 4)),
    "short_shape": header()[:30],
    "short_payload": header() + PAYLOAD[:-4],
    "trailing": header() + PAYLOAD + b"\x00",
    "huge_shape": header(dims=(1 << 21, 1 << 20, 1)),
    "overflow": header(dims=(1 << 40, 1 << 40, 1 << 40)),
}


@pytest.mark.parametrize("case", sorted(MALFORMED))
def test_header_errors_match_reference(ref, lib, tmp_path, case):
    p = tmp_path / f"{case}.pbst"
    p.write_bytes(MALFORMED[case])
    with pytest.raises(OracleError) as e:
        ref.read_tensor(p)
    rc, msg = info(lib, p)
    assert rc == e.value.code == 3
    assert msg == str(e.value)


def test_missing_file_matches_reference(ref, lib, tmp_path):
    p = tmp_path / "nope.pbst"
    with pytest.raises(OracleError) as e:
        ref.read_tensor(p)
    rc, msg = info(lib, p)
    assert rc == e.value.code == 3 and msg == str(e.value)


# ---- device payloads --------------------------------------------------------
gpu = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2510_21270_b200 import ops
    return ops


@gpu
@pytest.mark.parametrize("fdt", [np.float32, np.float64])
def test_load_reference_file(ops, ref, tmp_path, fdt):
    import torch
    rng = np.random.default_rng(5)
    a = (rng.standard_normal((3, 257, 128)) * 4).astype(fdt)
    ref.write_tensor(tmp_path / "a.pbst", a)
    t32 = ops.load_tensor(tmp_path / "a.pbst", dtype=torch.float32)
    np.testing.assert_array_equal(t32.cpu().numpy(), a.astype(np.float32))
    tb = ops.load_tensor(tmp_path / "a.pbst", dtype=torch.bfloat16)
    want = torch.from_numpy(a.astype(np.float32)).to(torch.bfloat16)
    assert torch.equal(tb.cpu(), want)
    m = a[0]
    ref.write_tensor(tmp_path / "m.pbst", m)
    t = ops.load_tensor(tmp_path / "m.pbst", dtype=torch.float32)
    assert t.shape == (257, 128)
    np.testing.assert_array_equal(t.cpu().numpy(), m.astype(np.float32))


@gpu
@pytest.mark.parametrize("src", ["f32", "bf16"])
@pytest.mark.parametrize("file_dtype", ["f32", "f64"])
def test_save_then_reference_reads(ops, ref, tmp_path, src, file_dtype):
    import torch
    g = torch.Generator(device="cuda").manual_seed(7)
    t = torch.randn(4, 300, 64, device="cuda", generator=g)
    if src == "bf16":
        t = t.to(torch.bfloat16)
    ops.save_tensor(tmp_path / "o.pbst", t, file_dtype=file_dtype)
    vals, fdt, nd = ref.read_tensor(tmp_path / "o.pbst")
    assert (fdt, nd) == ({"f32": 0, "f64": 1}[file_dtype], 3)
    np.testing.assert_array_equal(vals, t.float().cpu().numpy().astype(np.float64))
    ops.save_tensor(tmp_path / "m.pbst", t[1], file_dtype=file_dtype)
    vals, _, nd = ref.read_tensor(tmp_path / "m.pbst")
    assert nd == 2
    np.testing.assert_array_equal(vals, t[1].float().cpu().numpy().astype(np.float64))
    with pytest.raises(Exception, match="E_SHAPE: write_tensor: multiple heads require a 3-D stack"):
        ops.save_tensor(tmp_path / "x.pbst", t, as_stack=False)


@gpu
def test_multi_chunk_roundtrip(ops, tmp_path):
    import torch
    # 3 x 2048 x 4096 f32 = 96 MiB: two 64 MiB staging chunks each way
    t = torch.randn(3, 2048, 4096, device="cuda")
    ops.save_tensor(tmp_path / "big.pbst", t)
    assert os.path.getsize(tmp_path / "big.pbst") == 40 + t.numel() * 4
    back = ops.load_tensor(tmp_path / "big.pbst", dtype=torch.float32)
    assert torch.equal(back, t)


@gpu
@pytest.mark.parametrize("fdt", [np.float32, np.float64])
def test_non_finite_payload_matches_reference(ops, ref, tmp_path, fdt):
    import torch
    a = np.ones((2, 50, 16), dtype=fdt)
    a[1, 3, 5] = np.nan
    a[1, 40, 0] = np.inf
    p = tmp_path / "nan.pbst"
    ref.write_tensor(p, a)
    with pytest.raises(OracleError) as e:
        ref.read_tensor(p)
    with pytest.raises(Exception) as mine:
        ops.load_tensor(p, dtype=torch.float32)
    assert str(mine.value) == str(e.value)
    assert "E_FORMAT: non-finite element in tensor payload (byte offset" in str(mine.value)


# ---- run manifests (manifest.hpp) ----------------------------------------------
def _manifest(tmp_path, j):
    import json
    p = tmp_path / "run.json"
    p.write_text(json.dumps(j))
    return p


GOOD = {"inputs": {"q": "q.pbst", "k": "k.pbst", "v": "v.pbst"},
        "pipeline": {"block_size": 64, "segment_size": 128, "tau": 0.8, "strategy": "key_permute",
                     "precision": "f32"},
        "outputs": {"attention": "o.pbst", "report": "r.json"}}


def test_manifest_parse_and_defaults(tmp_path):
    from paper_2510_21270_b200 import manifest
    m = manifest.load_manifest(_manifest(tmp_path, GOOD))
    assert (m.block_size, m.segment_size, m.tau, m.strategy, m.precision) == (64, 128, 0.8, "key_permute", "f32")
    m = manifest.load_manifest(_manifest(tmp_path, {"inputs": GOOD["inputs"]}))
    # PipelineConfig / ForcedPolicy defaults (pipeline.hpp:30-37, block_selection.hpp:163-166)
    assert (m.block_size, m.segment_size, m.tau, m.strategy, m.precision, m.force_first_block,
            m.force_diagonal_band, m.scale, m.attention, m.report) == (128, 256, 0.9, "key_permute", "f64", True,
                                                                       True, 0.0, "", "")


@pytest.mark.parametrize("j,msg", [
    ({**GOOD, "extra": 1}, 'E_CONFIG: unknown key "extra" in manifest'),
    ({"pipeline": {}}, 'E_CONFIG: manifest needs exactly one of "workload" or "inputs"'),
    ({"inputs": {"q": "a", "k": "b"}}, "E_CONFIG: inputs need all of q, k, v paths"),
    ({"inputs": {"q": "a", "k": "b", "v": "c", "w": "d"}}, 'E_CONFIG: unknown key "w" in inputs'),
    ({"inputs": GOOD["inputs"], "pipeline": {"tau": "x"}}, 'E_CONFIG: bad value for "tau"'),
    ({"inputs": GOOD["inputs"], "pipeline": {"strategy": "zig"}}, "E_CONFIG: unknown permutation strategy 'zig'"),
    ({"inputs": GOOD["inputs"], "outputs": {"log": "x"}}, 'E_CONFIG: unknown key "log" in outputs'),
])
def test_manifest_errors(tmp_path, j, msg):
    from paper_2510_21270_b200 import _lib, manifest
    with pytest.raises(_lib.ConfigError) as e:
        manifest.load_manifest(_manifest(tmp_path, j))
    assert str(e.value) == msg


@gpu
def test_manifest_run_matches_reference(ops, ref, tmp_path):
    import json

    import oracle as orc
    from paper_2510_21270_b200 import manifest
    rng = np.random.default_rng(11)
    n, d, heads = 1024, 64, 2
    qkv = [rng.standard_normal((heads, n, d)) for _ in range(3)]
    qkv[1][:, ::97] += 6.0  # a few strong keys: a sparse selection
    # bf16-representable values, so the device (bf16) and the reference (f64 file) see the same numbers
    import torch
    qkv = [torch.from_numpy(x).to(torch.bfloat16).double().numpy() for x in qkv]
    for name, x in zip("qkv", qkv):
        ref.write_tensor(tmp_path / f"{name}.pbst", x)
    doc = manifest.run_manifest(manifest.load_manifest(_manifest(tmp_path, GOOD)), str(tmp_path))
    assert json.loads((tmp_path / "r.json").read_text()) == doc
    out, fdt, nd = ref.read_tensor(tmp_path / "o.pbst")
    assert (fdt, nd, out.shape) == (0, 3, (heads, n, d))
    cfg = orc.make_config(block_size=64, segment_size=128, tau=0.8, strategy="key_permute")
    o = Oracle("oracle")
    sel = adm = 0
    for h in range(heads):
        r = o.pbs_attention(qkv[0][h].astype(np.float32), qkv[1][h].astype(np.float32),
                            qkv[2][h].astype(np.float32), cfg)
        assert doc["heads"][h]["selected_blocks"] == r.report["selected_blocks"]
        assert doc["heads"][h]["total_admissible_blocks"] == r.report["total_admissible_blocks"]
        assert abs(doc["heads"][h]["block_density"] - r.report["block_density"]) < 1e-12
        # precision f32: the device's f32 path -- the reference's f32 arithmetic
        np.testing.assert_allclose(out[h], r.output, atol=1e-4)
        assert 0.8 <= doc["heads"][h]["attention_coverage"] <= 1.0
        sel += r.report["selected_blocks"]
        adm += r.report["total_admissible_blocks"]
    agg = doc["aggregate"]
    assert agg["selected_blocks"] == sel and agg["total_admissible_blocks"] == adm
    assert set(agg) == {"block_density", "causal_density_baseline", "attention_coverage", "selected_blocks",
                        "total_admissible_blocks", "timings_us"}


@gpu
def test_manifest_sweep_csv(ops, ref, tmp_path):
    import torch

    import oracle as orc
    from paper_2510_21270_b200 import manifest
    rng = np.random.default_rng(12)
    n, d = 1024, 64
    qkv = [torch.from_numpy(rng.standard_normal((1, n, d))).to(torch.bfloat16).double().numpy() for _ in range(3)]
    qkv[1][:, ::61] += 5.0
    for name, x in zip("qkv", qkv):
        ref.write_tensor(tmp_path / f"{name}.pbst", x)
    m = manifest.load_manifest(_manifest(tmp_path, GOOD))
    text = manifest.sweep_manifest(m, str(tmp_path), taus=[0.9, 0.5], segments=[128],
                                   strategies=["none", "key_permute", "none"], out_path=str(tmp_path / "s.csv"))
    assert (tmp_path / "s.csv").read_text() == text
    lines = text.splitlines()
    assert lines[0] == "tau,S,strategy,density,coverage,max_err,mean_err,time_us"
    rows = [ln.split(",") for ln in lines[1:]]
    assert [(r[0], r[1], r[2]) for r in rows] == [("0.5", "128", "key_permute"), ("0.9", "128", "key_permute"),
                                                  ("0.5", "128", "none"), ("0.9", "128", "none")]
    o = Oracle("oracle")
    for r in rows:
        cfg = orc.make_config(block_size=64, segment_size=128, tau=float(r[0]), strategy=r[2])
        want = o.pbs_attention(*(x[0].astype(np.float32) for x in qkv), cfg).report["block_density"]
        assert r[3] == "%.6f" % want
        # coverage in (0, 1]; errors against dense causal attention (large at low tau)
        assert 0.0 < float(r[4]) <= 1.0 and float(r[5]) >= float(r[6]) >= 0.0


def test_manifest_f64_needs_an_explicit_device_precision(tmp_path):
    """The device has no f64 path: an f64 manifest (the reference default) is
    refused with E_CONFIG unless the caller picks f32 / bf16."""
    import torch

    from paper_2510_21270_b200 import _lib, manifest
    m = manifest.load_manifest(_manifest(tmp_path, {"inputs": GOOD["inputs"]}))
    assert m.precision == "f64"
    with pytest.raises(_lib.ConfigError, match="E_CONFIG: precision f64 is not supported"):
        manifest.device_dtype(m)
    assert manifest.device_dtype(m, "f32") == torch.float32
    assert manifest.device_dtype(m, "bf16") == torch.bfloat16
    m32 = manifest.load_manifest(_manifest(tmp_path, GOOD))
    assert manifest.device_dtype(m32) == torch.float32
