"""The synthetic workload generator (workload.hpp:145-198, rng.hpp) in the
product library (pbs_generate_workload_head, host code) against the compiled
reference generator: every element bit for bit, every kind, both line
placements and precisions; validation texts of WorkloadSpec::validate; and
`workload` run manifests (manifest.hpp:26-39) through the device path against
the reference pipeline on the reference-generated tensors."""
import json

import numpy as np
import pytest

from conftest import assert_f32

KINDS = ("gaussian", "vertical_lines", "block_diag", "mixed")


@pytest.fixture(scope="module")
def ops():
    from paper_2510_21270_b200 import ops as _ops
    _ops.lib()  # host entry points work without a GPU
    return _ops


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("scatter", ["clustered", "scattered"])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_generator_bit_identical_to_reference(ops, ref, kind, scatter, prec):
    from oracle.gen_golden import generate_head
    n, d, seed, lines, strength = 777, 48, 12345678901, 9, 40.0
    spec = ops.workload_spec(kind=kind, n=n, d=d, heads=3, seed=seed, line_count=lines, line_strength=strength,
                             scatter=scatter)
    dt = np.float32 if prec == "f32" else np.float64
    for head in (0, 2):
        q, k, v, planted = ops.generate_workload_head(spec, head, 64, 256, prec)
        rq, rk, rv, rp = generate_head(ref, kind, n, d, seed, 64, 256, head=head, line_count=lines,
                                       line_strength=strength, scatter=int(scatter == "scattered"), dtype=dt)
        for a, b in ((q, rq), (k, rk), (v, rv)):
            assert a.dtype == b.dtype and np.array_equal(a.view(np.uint8), b.view(np.uint8))
        np.testing.assert_array_equal(planted, rp)


@pytest.mark.parametrize("block,segment", [(128, 256), (64, 0), (256, 128), (16, 4096)])
def test_line_placement_variants(ops, ref, block, segment):
    """plan_line_positions' branches: segmented, no segmentation, S < B, more lines than segments."""
    from oracle.gen_golden import generate_head
    spec = ops.workload_spec(kind="vertical_lines", n=2000, d=8, seed=3, line_count=37, line_strength=5.0)
    q, k, v, planted = ops.generate_workload_head(spec, 0, block, segment, "f64")
    rq, rk, rv, rp = generate_head(ref, "vertical_lines", 2000, 8, 3, block, segment, line_count=37,
                                   line_strength=5.0, scatter=1, dtype=np.float64)
    np.testing.assert_array_equal(planted, rp)
    assert np.array_equal(k.view(np.uint8), rk.view(np.uint8))


@pytest.mark.parametrize("kw,msg", [
    (dict(n=0), "E_CONFIG: workload dims must be >= 1"),
    (dict(kind="vertical_lines", n=10, line_count=11), "E_CONFIG: line count exceeds sequence length"),
    (dict(kind="mixed", line_strength=0.0), "E_CONFIG: line strength must be > 0"),
])
def test_generator_validation(ops, kw, msg):
    from paper_2510_21270_b200 import _lib
    with pytest.raises(_lib.ConfigError) as e:
        ops.generate_workload_head(ops.workload_spec(**kw), 0, 64, 256, "f32")
    assert str(e.value) == msg


def _manifest(tmp_path, j):
    p = tmp_path / "m.json"
    p.write_text(json.dumps(j))
    return str(p)


def test_workload_manifest_parse(tmp_path):
    from paper_2510_21270_b200 import _lib, manifest
    m = manifest.load_manifest(_manifest(tmp_path, {"workload": {"kind": "mixed", "n": 512, "heads": 2}}))
    assert m.workload == {"kind": "mixed", "n": 512, "d": 64, "heads": 2, "seed": 0, "line_count": 8,
                          "line_strength": 150.0, "scatter": "scattered"}
    for j, msg in (({"workload": {"kind": "zig"}}, "E_CONFIG: unknown workload kind 'zig'"),
                   ({"workload": {"scatter": "x"}}, "E_CONFIG: unknown scatter mode 'x'"),
                   ({"workload": {"heads": 0}}, "E_CONFIG: workload dims must be >= 1"),
                   ({"workload": {"n": 4, "kind": "vertical_lines"}}, "E_CONFIG: line count exceeds sequence length"),
                   ({"workload": {"seed": -1}}, 'E_CONFIG: bad value for "seed"'),
                   ({"workload": {"lines": 3}}, 'E_CONFIG: unknown key "lines" in workload'),
                   ({"workload": {}, "inputs": {"q": "a", "k": "b", "v": "c"}},
                    'E_CONFIG: manifest needs exactly one of "workload" or "inputs"')):
        with pytest.raises(_lib.ConfigError) as e:
            manifest.load_manifest(_manifest(tmp_path, j))
        assert str(e.value) == msg


@pytest.mark.gpu
def test_workload_manifest_run_matches_reference(ops, ref, tmp_path):
    """pbs_main.cpp `run` on a workload manifest: the reference generates the same
    tensors (f32) and runs its pipeline per head; counts, densities and the
    output file agree (f32 bar), and --seed overrides the workload seed."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import make_config
    from oracle.gen_golden import generate_head
    from paper_2510_21270_b200 import manifest
    w = {"kind": "vertical_lines", "n": 2048, "d": 64, "heads": 2, "seed": 7, "line_count": 16,
         "line_strength": 150.0}
    j = {"workload": w, "pipeline": {"block_size": 64, "segment_size": 128, "tau": 0.9, "precision": "f32"},
         "outputs": {"attention": "o.pbst", "report": "r.json"}}
    path = _manifest(tmp_path, j)
    assert manifest.main(["run", "--manifest", path, "--seed", "11"]) == 0
    doc = json.loads((tmp_path / "r.json").read_text())
    out, fdt, nd = ref.read_tensor(tmp_path / "o.pbst")
    assert (fdt, nd, out.shape) == (0, 3, (2, 2048, 64))
    cfg = make_config(block_size=64, segment_size=128, tau=0.9, strategy="key_permute")
    for h in range(2):
        q, k, v, _ = generate_head(ref, "vertical_lines", 2048, 64, 11, 64, 128, head=h, line_count=16,
                                   line_strength=150.0, scatter=1, dtype=np.float32)
        r = ref.pbs_attention(q, k, v, cfg)
        for key in ("selected_blocks", "total_admissible_blocks", "block_density", "causal_density_baseline"):
            assert doc["heads"][h][key] == r.report[key], key
        assert_f32(np.abs(out[h] - r.output))
