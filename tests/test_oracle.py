"""Pin the CPU oracle (oracle/pbs_oracle.c) before it is trusted as the checker.

Three kinds of pins, all CPU-only:
  1. the reference's own golden files and known-answer tests, re-expressed
     (citations point into /root/reference/proj/tests/unit/*.cpp);
  2. the committed reference-generated fixtures tests/golden/ref_pipeline_f32_*
     (oracle/gen_golden.py ran the compiled reference to make them);
  3. when oracle/_ref/libpbsref.so is present, bit-for-bit agreement with the
     unmodified reference headers on randomised inputs.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import OracleError, inverse, make_config

F32, F64 = np.float32, np.float64


def bf16_round(x):
    """Round-to-nearest-even to bf16, returned as float32 (exact upcast)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


# --------------------------------------------------------------------------
# 1. golden files
# --------------------------------------------------------------------------
def test_golden_run256(oracle):
    """pipeline_test.cpp:79-103 (GoldenRun256) against tests/golden/pipeline256.json."""
    g = np.load(os.path.join(GOLDEN, "pipeline256.npz"))
    want = json.load(open(os.path.join(GOLDEN, "pipeline256.json")))
    cfg = make_config(block_size=32, segment_size=64, tau=0.9, strategy="key_permute")
    res = oracle.pbs_attention(g["q"], g["k"], g["v"], cfg)
    ref_out = oracle.attention_oracle(g["q"], g["k"], g["v"], block_size=32, causal=True)
    diff = np.abs(res.output - ref_out)
    assert abs(diff.max() - want["max_err"]) <= 1e-9
    assert abs(diff.mean() - want["mean_err"]) <= 1e-9
    assert res.report["block_density"] == want["density"]


def test_golden_attn4(oracle):
    """attention_test.cpp:50-73: oracle full/causal vs the NumPy f64 goldens (make_golden.py)."""
    g = np.load(os.path.join(GOLDEN, "attn4.npz"))
    full = oracle.attention_oracle(g["q"], g["k"], g["v"], block_size=1, causal=False)
    causal = oracle.attention_oracle(g["q"], g["k"], g["v"], block_size=1, causal=True)
    assert np.max(np.abs(full - g["expected_full"])) <= 1e-12
    assert np.max(np.abs(causal - g["expected_causal"])) <= 1e-12


@pytest.mark.parametrize("kind", ["vertical_lines", "mixed", "gaussian"])
def test_reference_fixtures(oracle, kind):
    """Bit-exact agreement with reference runs recorded by oracle/gen_golden.py."""
    g = np.load(os.path.join(GOLDEN, f"ref_pipeline_f32_{kind}.npz"))
    meta = json.load(open(os.path.join(GOLDEN, "ref_pipeline_f32.json")))[kind]
    cfg = make_config(block_size=meta["block"], segment_size=meta["segment"], tau=meta["tau"],
                      strategy=meta["strategy"])
    res = oracle.pbs_attention(g["q"], g["k"], g["v"], cfg)
    np.testing.assert_array_equal(res.sigma, g["sigma"])
    np.testing.assert_array_equal(res.pi, g["pi"])
    np.testing.assert_array_equal(res.mask, g["mask"])
    np.testing.assert_array_equal(res.output, g["output"])
    for key, val in meta["report"].items():
        assert res.report[key] == val, key
    imp, _ = oracle.estimate_key_importance(g["q"], g["k"], meta["block"])
    np.testing.assert_array_equal(imp, g["importance"])
    t = g["mask"].shape[0]
    causal = oracle.build_block_causal_mask(t, meta["block"], meta["segment"])
    scores = oracle.meanpool_block_scores(g["q"][res.sigma], g["k"][res.pi], meta["block"], causal)
    np.testing.assert_array_equal(scores, g["block_scores"])


# --------------------------------------------------------------------------
# 2. known-answer tests of the reference unit suites
# --------------------------------------------------------------------------
def test_argsort_with_ties_kat(oracle):
    """permutation_test.cpp:178-184."""
    s = np.array([.1, .4, .2, .3, .05, .05, .6, .3], dtype=F64)
    perm = oracle.build_key_permutation(s, 4)
    np.testing.assert_array_equal(perm, [1, 3, 2, 0, 4 + 2, 4 + 3, 4 + 0, 4 + 1])


def test_singleton_and_oversized_segments(oracle):
    """permutation_test.cpp:166-176."""
    s = np.array([0.5, 0.1, 0.4], dtype=F64)
    np.testing.assert_array_equal(oracle.build_key_permutation(s, 1), [0, 1, 2])
    np.testing.assert_array_equal(oracle.build_key_permutation(s, 7), [0, 1, 2])


def test_remainder_identity_and_nonincreasing(oracle):
    """permutation_test.cpp:67-94, 186-199."""
    rng = np.random.default_rng(9)
    for _ in range(20):
        n = int(rng.integers(1, 65))
        s = int(rng.integers(1, 17))
        scores = rng.random(n)
        perm = oracle.build_key_permutation(scores, s)
        g = n // s
        np.testing.assert_array_equal(perm[g * s:], np.arange(g * s, n))
        for seg in range(g):
            blk = perm[seg * s:(seg + 1) * s]
            assert sorted(blk) == list(range(seg * s, (seg + 1) * s))
            assert np.all(np.diff(scores[blk]) <= 0)


def test_query_permutation_kats(oracle):
    """permutation_test.cpp:201-234."""
    k = np.array([[1, 0], [1, 0], [0, 1], [0, 1]], dtype=F64)
    q = np.array([[0, 2], [3, 0], [0, 1], [2, 0.1]], dtype=F64)
    np.testing.assert_array_equal(oracle.build_query_permutation(q, k, 2, 4), [1, 3, 0, 2])
    q0 = np.array([[0, 0], [1, 0], [0, 1], [1, 0]], dtype=F64)
    np.testing.assert_array_equal(oracle.build_query_permutation(q0, k, 2, 4), [1, 3, 2, 0])
    rng = np.random.default_rng(10)
    q8, k8 = rng.standard_normal((8, 4)), rng.standard_normal((8, 4))
    np.testing.assert_array_equal(oracle.build_query_permutation(q8, k8, 8, 8), np.arange(8))
    np.testing.assert_array_equal(oracle.build_query_permutation(q8, k8, 2, 1), np.arange(8))


def test_importance_kats(oracle):
    """permutation_test.cpp:96-164: uniform, dominant key, sums to one, N < B."""
    rng = np.random.default_rng(3)
    q = np.zeros((16, 4))
    k = rng.standard_normal((16, 4))
    imp, src = oracle.estimate_key_importance(q, k, 4)
    np.testing.assert_allclose(imp, 1 / 16, rtol=0, atol=1e-15)
    assert src == 3
    q = rng.standard_normal((10, 4))
    k = rng.standard_normal((10, 4))
    k[7] = 50 * q[-4:].mean(axis=0)
    imp, _ = oracle.estimate_key_importance(q, k, 4)
    assert int(np.argmax(imp)) == 7
    assert abs(imp.sum() - 1) <= 1e-12
    imp, src = oracle.estimate_key_importance(q[:3], k, 8)  # N < B: all queries
    assert src == 0 and abs(imp.sum() - 1) <= 1e-12


def test_block_causal_mask_counts(oracle):
    """block_selection_test.cpp:27-48."""
    c = oracle.build_block_causal_mask(4, 128, 0, dtype=F64)
    assert (c == 0).sum() == 10
    c = oracle.build_block_causal_mask(4, 128, 256, dtype=F64)
    assert c[0, 1] == 0 and c[0, 2] == -np.inf and c[2, 3] == 0
    assert (c == 0).sum() == 12


def test_pooled_softmax_kat(oracle):
    """block_selection_test.cpp:73-102 at 1e-14."""
    q = np.array([[1, 0], [0, 2], [1, 1], [2, 0], [0, 1], [1, 2], [2, 1], [0, 0]], dtype=F64)
    k = np.array([[0, 1], [1, 1], [2, 0], [1, 0], [0, 2], [2, 2], [1, 2], [2, 1]], dtype=F64)
    causal = oracle.build_block_causal_mask(4, 2, 0, dtype=F64)
    s = oracle.meanpool_block_scores(q, k, 2, causal)
    qb = q.reshape(4, 2, 2).mean(axis=1)
    kb = k.reshape(4, 2, 2).mean(axis=1)
    lg = qb @ kb.T / np.sqrt(2)
    lg = np.where(np.tril(np.ones((4, 4))) > 0, lg, -np.inf)
    w = np.exp(lg - lg.max(axis=1, keepdims=True))
    w /= w.sum(axis=1, keepdims=True)
    assert np.max(np.abs(s - w)) <= 1e-14


def test_short_final_block(oracle):
    """block_selection_test.cpp:104-119."""
    q = np.arange(1, 6, dtype=F64)[:, None]
    k = np.ones((5, 1))
    causal = oracle.build_block_causal_mask(3, 2, 0, dtype=F64)
    s = oracle.meanpool_block_scores(q, k, 2, causal)
    for i in range(3):
        np.testing.assert_allclose(s[i, :i + 1], 1 / (i + 1), atol=1e-12)


def _scores(rows, b, s, oracle):
    t = len(rows)
    causal = oracle.build_block_causal_mask(t, b, s, dtype=F64)
    sc = np.where(causal == 0, np.array(rows, dtype=F64), 0.0)
    return sc, causal


def test_select_tau_zero_kat(oracle):
    """block_selection_test.cpp:135-153."""
    sc, causal = _scores([[1.0, 0, 0, 0], [0.3, 0.7, 0, 0], [0.2, 0.5, 0.3, 0], [0.1, 0.2, 0.3, 0.4]],
                         4, 0, oracle)
    m = oracle.select_blocks(sc, causal, 4, 0, 0.0)
    assert m[0, 0] and m[1, 1] and m[1, 0] and m[2, 1] and m[2, 0] and m[2, 2]
    assert not m[3, 1] and m[3, 3] and m[3, 0] and not m[3, 2]


def test_select_brute_force_and_monotone(oracle):
    """block_selection_test.cpp:155-231 (tau=1, minimal prefix, monotone)."""
    rng = np.random.default_rng(44)
    for _ in range(50):
        t = int(rng.integers(1, 11))
        rows = np.zeros((t, t))
        for i in range(t):
            rows[i, :i + 1] = rng.random(i + 1)
            rows[i, :i + 1] /= rows[i, :i + 1].sum()
        sc, causal = _scores(rows, 4, 0, oracle)
        tau = float(rng.random())
        m = oracle.select_blocks(sc, causal, 4, 0, tau, False, False)
        for i in range(t):
            order = sorted(range(i + 1), key=lambda j: (-rows[i, j], j))
            cum, want = 0.0, []
            for j in order:
                want.append(j)
                cum += rows[i, j]
                if cum >= tau:
                    break
            assert m[i].sum() == len(want)
            assert all(m[i, j] for j in want)
        full = oracle.select_blocks(sc, causal, 4, 0, 1.0)
        np.testing.assert_array_equal(full, np.tril(np.ones((t, t), dtype=np.uint8)))
        t1, t2 = sorted(rng.random(2))
        lo = oracle.select_blocks(sc, causal, 4, 0, float(t1))
        hi = oracle.select_blocks(sc, causal, 4, 0, float(t2))
        assert np.all(hi[lo > 0] > 0)


def test_select_top_k_brute_force(oracle):
    """The top-k extension (no reference counterpart): the first k blocks of
    the reference's stable descending order (ties by ascending index) + forced."""
    rng = np.random.default_rng(45)
    for _ in range(40):
        t = int(rng.integers(1, 12))
        rows = np.zeros((t, t))
        for i in range(t):
            rows[i, :i + 1] = np.round(rng.random(i + 1), 1)  # rounded: plenty of ties
        sc, causal = _scores(rows, 4, 0, oracle)
        k = int(rng.integers(1, 6))
        m = oracle.select_blocks(sc, causal, 4, 0, 0.9, False, False, top_k=k)
        for i in range(t):
            order = sorted(range(i + 1), key=lambda j: (-sc[i, j], j))
            want = set(order[:k])
            assert set(np.flatnonzero(m[i])) == want
    rows = np.array([[1.0, 0, 0, 0], [0.1, 0.5, 0, 0], [0.1, 0.2, 0.2, 0], [0.2, 0.2, 0.3, 0.3]])
    sc, causal = _scores(rows, 4, 0, oracle)
    m = oracle.select_blocks(sc, causal, 4, 0, 0.9, True, False, top_k=2)
    np.testing.assert_array_equal(m, [[1, 0, 0, 0], [1, 1, 0, 0], [1, 1, 1, 0], [1, 0, 1, 1]])


def test_select_forced_band(oracle):
    """block_selection_test.cpp:233-252."""
    rows = np.zeros((8, 8))
    rows[:, 0] = 1.0
    sc, causal = _scores(rows, 32, 64, oracle)
    m = oracle.select_blocks(sc, causal, 32, 64, 0.0)
    for i in range(8):
        assert m[i, 0]
        for j in range(8):
            if j // 2 == i // 2:
                assert m[i, j]
            assert not (m[i, j] and j // 2 > i // 2)


def test_sparse_full_mask_equals_tiled_bitwise(oracle):
    """attention_test.cpp:125-138 / acceptance C3: a full mask is the tiled path."""
    rng = np.random.default_rng(5)
    q, k, v = (rng.standard_normal((37, 6)).astype(F32) for _ in range(3))
    a = oracle.attention_block_sparse(q, k, v, 8, mask=np.ones((5, 5), np.uint8))
    b = oracle.attention_block_sparse(q, k, v, 8)
    np.testing.assert_array_equal(a, b)
    ref = oracle.attention_oracle(q.astype(F64), k.astype(F64), v.astype(F64), 8)
    assert np.max(np.abs(a - ref)) <= 1e-5


def test_degenerate_row(oracle):
    """attention_test.cpp:261-282: an all-masked row raises E_DEGENERATE with its block id."""
    rng = np.random.default_rng(6)
    q, k, v = (rng.standard_normal((16, 4)) for _ in range(3))
    mask = np.zeros((4, 4), np.uint8)
    mask[0, 0] = 1
    with pytest.raises(OracleError) as e:
        oracle.attention_block_sparse(q, k, v, 4, mask=mask)
    assert e.value.code == 5 and e.value.query_block == 1
    assert "E_DEGENERATE" in str(e.value)


def test_pipeline_tau_one_exact(oracle):
    """pipeline_test.cpp:27-58 (C4): tau=1 is the causal oracle for every strategy."""
    rng = np.random.default_rng(51)
    q, k, v = (rng.standard_normal((96, 8)) for _ in range(3))
    want = oracle.attention_oracle(q, k, v, 16, causal=True)
    for strategy in ["none", "key_permute", "query_permute", "both"]:
        for s in (16, 32, 64):
            cfg = make_config(block_size=16, segment_size=s, tau=1.0, strategy=strategy)
            res = oracle.pbs_attention(q, k, v, cfg)
            assert np.max(np.abs(res.output - want)) <= 1e-10, (strategy, s)


def test_pipeline_causality_bitwise(oracle):
    """pipeline_test.cpp:105-128 (C5)."""
    rng = np.random.default_rng(53)
    q, k, v = (rng.standard_normal((64, 4)) for _ in range(3))
    cfg = make_config(block_size=8, segment_size=16, tau=0.8)
    base = oracle.pbs_attention(q, k, v, cfg).output
    for j in (5, 20, 63):
        v2 = v.copy()
        v2[j] += 100.0
        out = oracle.pbs_attention(q, k, v2, cfg).output
        np.testing.assert_array_equal(out[:j], base[:j])


def test_config_validation(oracle):
    """pipeline_test.cpp:244-270: bad configs are E_CONFIG (exit code 2)."""
    q = np.zeros((8, 2))
    for cfg in (make_config(block_size=0), make_config(block_size=4, segment_size=6),
                make_config(block_size=4, segment_size=2), make_config(block_size=4, tau=1.5),
                make_config(block_size=4, segment_size=0, strategy="key_permute"),
                make_config(block_size=4, segment_size=8, scale=-1.0)):
        with pytest.raises(OracleError) as e:
            oracle.pbs_attention(q, q, q, cfg)
        assert e.value.code == 2


def test_segment_equal_block_gives_causal_density(oracle):
    """pipeline_test.cpp:313-329: S == B with tau=1 selects exactly the causal grid."""
    rng = np.random.default_rng(60)
    q, k, v = (rng.standard_normal((64, 4)) for _ in range(3))
    res = oracle.pbs_attention(q, k, v, make_config(block_size=8, segment_size=8, tau=1.0))
    assert res.report["block_density"] == res.report["causal_density_baseline"]


# --------------------------------------------------------------------------
# 3. bit-for-bit against the compiled reference headers
# --------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", [F32, F64])
@pytest.mark.parametrize("seed", range(4))
def test_stagewise_matches_reference(oracle, ref, dtype, seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(20, 200))
    d = int(rng.integers(1, 24))
    b = int(rng.choice([1, 4, 8, 16]))
    s = b * int(rng.integers(1, 5))
    q = rng.standard_normal((n, d)).astype(dtype)
    k = rng.standard_normal((n, d)).astype(dtype)
    v = rng.standard_normal((n, d)).astype(dtype)
    if seed % 2:  # bf16-origin data, the GPU path's inputs
        q, k, v = (bf16_round(x).astype(dtype) for x in (q, k, v))
    imp_o, src_o = oracle.estimate_key_importance(q, k, b)
    imp_r, src_r = ref.estimate_key_importance(q, k, b)
    np.testing.assert_array_equal(imp_o, imp_r)
    assert src_o == src_r
    np.testing.assert_array_equal(oracle.build_key_permutation(imp_o, s),
                                  ref.build_key_permutation(imp_r, s))
    np.testing.assert_array_equal(oracle.build_query_permutation(q, k, b, s),
                                  ref.build_query_permutation(q, k, b, s))
    t = (n + b - 1) // b
    c_o = oracle.build_block_causal_mask(t, b, s, dtype=dtype)
    np.testing.assert_array_equal(c_o, ref.build_block_causal_mask(t, b, s, dtype=dtype))
    sc_o = oracle.meanpool_block_scores(q, k, b, c_o)
    sc_r = ref.meanpool_block_scores(q, k, b, c_o)
    np.testing.assert_array_equal(sc_o, sc_r)
    tau = float(rng.random())
    np.testing.assert_array_equal(oracle.select_blocks(sc_o, c_o, b, s, tau),
                                  ref.select_blocks(sc_r, c_o, b, s, tau))
    mask = (rng.random((t, t)) < 0.6).astype(np.uint8)
    np.fill_diagonal(mask, 1)
    qo = rng.permutation(n).astype(np.int32)
    ko = rng.permutation(n).astype(np.int32)
    for args in (dict(), dict(causal=True), dict(q_orig=np.arange(n, dtype=np.int32), k_orig=ko)):
        try:
            a = oracle.attention_block_sparse(q, k, v, b, mask=mask, **args)
        except OracleError as e:
            with pytest.raises(OracleError) as e2:
                ref.attention_block_sparse(q, k, v, b, mask=mask, **args)
            assert e.code == e2.value.code and e.query_block == e2.value.query_block
            continue
        np.testing.assert_array_equal(a, ref.attention_block_sparse(q, k, v, b, mask=mask, **args))
    np.testing.assert_array_equal(
        oracle.attention_oracle(q, k, v, b, q_orig=qo, k_orig=ko),
        ref.attention_oracle(q, k, v, b, q_orig=qo, k_orig=ko))


@pytest.mark.parametrize("strategy", ["none", "key_permute", "query_permute", "both"])
@pytest.mark.parametrize("dtype", [F32, F64])
def test_pipeline_matches_reference(oracle, ref, strategy, dtype):
    rng = np.random.default_rng(7)
    for n, d, b, s, tau in ((130, 8, 8, 16, 0.5), (256, 16, 16, 64, 0.9), (77, 5, 4, 8, 0.3)):
        q, k, v = (bf16_round(rng.standard_normal((n, d))).astype(dtype) for _ in range(3))
        if strategy == "none":
            s = 0 if n % 2 else s
        cfg = make_config(block_size=b, segment_size=s, tau=tau, strategy=strategy)
        a = oracle.pbs_attention(q, k, v, cfg)
        r = ref.pbs_attention(q, k, v, cfg)
        np.testing.assert_array_equal(a.sigma, r.sigma)
        np.testing.assert_array_equal(a.pi, r.pi)
        np.testing.assert_array_equal(a.mask, r.mask)
        np.testing.assert_array_equal(a.output, r.output)
        for key in ("block_density", "causal_density_baseline", "pooled_score_coverage",
                    "selected_blocks", "total_admissible_blocks"):
            assert a.report[key] == r.report[key], key


def test_inverse_roundtrip():
    """permutation_test.cpp:18-65: p o p^-1 = id."""
    rng = np.random.default_rng(1)
    p = rng.permutation(100).astype(np.int32)
    inv = inverse(p)
    np.testing.assert_array_equal(p[inv], np.arange(100))
    np.testing.assert_array_equal(inv[p], np.arange(100))


@pytest.mark.parametrize("strategy", ["none", "key_permute", "query_permute", "both"])
@pytest.mark.parametrize("dtype", [F32, F64])
def test_attention_coverage_matches_reference(oracle, ref, strategy, dtype):
    """attention_coverage (pipeline.hpp:198-243): the C restatement equals the
    compiled reference bit for bit on the pipeline's own mask / sigma / pi."""
    rng = np.random.default_rng(17)
    for n, d, b, s, tau in ((130, 8, 8, 16, 0.5), (256, 16, 16, 64, 0.9)):
        q, k, v = (bf16_round(rng.standard_normal((n, d))).astype(dtype) for _ in range(3))
        if strategy == "none":
            s = 0
        cfg = make_config(block_size=b, segment_size=s, tau=tau, strategy=strategy)
        r = ref.pbs_attention(q, k, v, cfg)
        a = oracle.attention_coverage(q, k, r.mask, b, r.sigma, r.pi)
        want = ref.attention_coverage(q, k, r.mask, b, r.sigma, r.pi)
        assert a == want
        assert 0.0 < a <= 1.0


def test_attention_coverage_properties(oracle):
    """Full mask -> coverage 1; tau = 1 selects the whole causal grid (C4);
    a stricter tau never raises coverage (monotone, block_selection_test.cpp:211-231)."""
    rng = np.random.default_rng(3)
    n, d, b, s = 256, 16, 16, 64
    q, k, v = (rng.standard_normal((n, d)).astype(F64) for _ in range(3))
    t = n // b
    assert oracle.attention_coverage(q, k, np.ones((t, t), np.uint8), b) == pytest.approx(1.0, abs=1e-12)
    cov = []
    for tau in (0.3, 0.6, 0.9, 1.0):
        r = oracle.pbs_attention(q, k, v, make_config(block_size=b, segment_size=s, tau=tau))
        cov.append(oracle.attention_coverage(q, k, r.mask, b, r.sigma, r.pi))
    assert cov[-1] == pytest.approx(1.0, abs=1e-12)
    assert all(x <= y + 1e-12 for x, y in zip(cov, cov[1:]))
