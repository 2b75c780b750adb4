"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Bar:
  * bit-exact: importance scores, pi / sigma (+ inverses), block scores,
    masks, selected-block counts;
  * outputs: bf16 path vs the oracle run in fp32 on the bf16-upcast inputs,
    |err|max <= 2e-2 and mean <= 2e-3 (unit-Gaussian V); f32 path <= 1e-4.
The oracle itself is pinned by tests/test_oracle.py.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import BF16_MAX, BF16_MEAN, F32_MAX, assert_bf16, assert_f32  # noqa: E402


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2510_21270_b200 import ops as _ops

    _ops.lib()
    return _ops


def bf16_inputs(rng, hq, hkv, n, d, kind="gaussian", lines=8, strength=30.0, block=128, segment=256):
    """Synthetic Q/K/V (head-major) rounded to bf16; returns torch bf16 + numpy f32 upcasts."""
    q = rng.standard_normal((hq, n, d)).astype(np.float32)
    k = rng.standard_normal((hkv, n, d)).astype(np.float32)
    v = rng.standard_normal((hkv, n, d)).astype(np.float32)
    if kind == "vertical_lines":  # workload.hpp:182-194, one direction per kv head
        g = hq // hkv
        for kh in range(hkv):
            u = rng.standard_normal(d)
            u /= np.linalg.norm(u)
            q[kh * g:(kh + 1) * g] += np.sqrt(d) * u
            pos = rng.choice(n, size=min(lines, n), replace=False)
            k[kh, pos] += strength * u
    tq = torch.from_numpy(q).to(torch.bfloat16)
    tk = torch.from_numpy(k).to(torch.bfloat16)
    tv = torch.from_numpy(v).to(torch.bfloat16)
    return (tq.cuda(), tk.cuda(), tv.cuda(), tq.float().numpy(), tk.float().numpy(), tv.float().numpy())


def kv_of(h, hq, hkv):
    return h // (hq // hkv)


# ---------------------------------------------------------------------------
@pytest.mark.parametrize("hq,hkv,n,d,b,dtype", [
    (1, 1, 1024, 128, 128, "bf16"),
    (4, 2, 777, 64, 64, "bf16"),
    (2, 2, 300, 16, 16, "f32"),
    (1, 1, 50, 32, 64, "bf16"),   # N < B: all queries
    (1, 1, 4096, 128, 64, "f32"),  # config 1 (B=64)
    (2, 1, 1000, 64, 40, "bf16"),  # take % 32 != 0: cp.async denominators, 8-row chunk
    (1, 1, 700, 128, 96, "bf16"),  # three TMA row groups, ragged last key tile
])
def test_importance_and_key_permutation_bitexact(ops, oracle, hq, hkv, n, d, b, dtype):
    rng = np.random.default_rng(n + d)
    tq, tk, tv, q, k, v = bf16_inputs(rng, hq, hkv, n, d, kind="vertical_lines", block=b)
    if dtype == "f32":
        q = rng.standard_normal((hq, n, d)).astype(np.float32)
        k = rng.standard_normal((hkv, n, d)).astype(np.float32)
        tq, tk = torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda()
    scores = ops.estimate_key_importance(tq, tk, b).cpu().numpy()
    s = max(b, 4 * b) if n >= 4 * b else b
    perm, inv = ops.build_key_permutation(torch.from_numpy(scores).cuda(), s)
    perm, inv = perm.cpu().numpy(), inv.cpu().numpy()
    for h in range(hq):
        want, _ = oracle.estimate_key_importance(q[h], k[kv_of(h, hq, hkv)], b)
        np.testing.assert_array_equal(scores[h].view(np.uint32), want.view(np.uint32))
        wp = oracle.build_key_permutation(want, s)
        np.testing.assert_array_equal(perm[h], wp)
        np.testing.assert_array_equal(inv[h][perm[h]], np.arange(n))


def test_key_permutation_ties_kat(ops):
    """permutation_test.cpp:178-184 through the device sort."""
    s = torch.tensor([[.1, .4, .2, .3, .05, .05, .6, .3]], dtype=torch.float32).cuda()
    perm, inv = ops.build_key_permutation(s, 4)
    assert perm.cpu().tolist() == [[1, 3, 2, 0, 6, 7, 4, 5]]
    zeros = torch.zeros(1, 256 * 3 + 7, dtype=torch.float32).cuda()  # all ties + ragged tail
    perm, _ = ops.build_key_permutation(zeros, 256)
    assert perm.cpu().tolist()[0] == list(range(256 * 3 + 7))


@pytest.mark.parametrize("n,d,b,s,tau", [(2048, 128, 128, 256, 0.9), (1000, 64, 32, 64, 0.5),
                                         (640, 32, 64, 0, 0.7),
                                         # register sorts: 2, 8 and 16 keys per thread (T = 256 / 1024 / 2048)
                                         (4096, 32, 16, 64, 0.9), (8192, 16, 8, 32, 0.9),
                                         (16384, 16, 8, 64, 0.95)])
def test_block_scores_and_selection_bitexact(ops, oracle, n, d, b, s, tau):
    rng = np.random.default_rng(7)
    tq, tk, tv, q, k, v = bf16_inputs(rng, 2, 1, n, d, kind="vertical_lines")
    scores = ops.meanpool_block_scores(tq, tk, b, s).cpu().numpy()
    mask, kv_idx, kv_cnt = ops.select_blocks(torch.from_numpy(scores).cuda(), b, s, tau)
    mask, kv_idx, kv_cnt = mask.cpu().numpy(), kv_idx.cpu().numpy(), kv_cnt.cpu().numpy()
    t = -(-n // b)
    causal = oracle.build_block_causal_mask(t, b, s)
    for h in range(2):
        want = oracle.meanpool_block_scores(q[h], k[0], b, causal)
        np.testing.assert_array_equal(scores[h].view(np.uint32), want.view(np.uint32))
        wm = oracle.select_blocks(want, causal, b, s, tau)
        np.testing.assert_array_equal(mask[h], wm)
        for i in range(t):
            sel = np.flatnonzero(wm[i])
            assert kv_cnt[h, i] == sel.size
            np.testing.assert_array_equal(kv_idx[h, i, :sel.size], sel)


@pytest.mark.parametrize("strategy", ["key_permute", "none", "query_permute", "both"])
@pytest.mark.parametrize("hq,hkv,n,d,b,s,tau", [
    (2, 1, 1024, 128, 128, 256, 0.9),
    (4, 2, 1536 + 64, 128, 128, 256, 0.8),  # ragged final block
    (1, 1, 512, 64, 32, 128, 0.7),
    (2, 1, 1024, 128, 64, 256, 0.9),  # B = 64 on the tensor cores (2 x 2 blocks per tile)
    (4, 2, 2048 + 64 + 17, 128, 64, 128, 0.85),  # B = 64, ragged, lone last block of a tile pair
])
def test_pipeline_matches_oracle(ops, oracle, monkeypatch, strategy, hq, hkv, n, d, b, s, tau):
    from oracle import make_config as ocfg

    if d == 128:  # bf16, d = 128, B = 64 / 128: must run the tcgen05 kernel
        monkeypatch.setenv("PBS_REQUIRE_TC", "1")
    rng = np.random.default_rng(11)
    tq, tk, tv, q, k, v = bf16_inputs(rng, hq, hkv, n, d, kind="vertical_lines", strength=20.0, block=b)
    if strategy == "none":
        s = 0
    cfg = ops.make_config(block_size=b, segment_size=s, tau=tau, strategy=strategy)
    res = ops.pbs_attention(tq, tk, tv, cfg)
    out = res.output.float().cpu().numpy()
    sigma, pi, mask = res.sigma.cpu().numpy(), res.pi.cpu().numpy(), res.mask.cpu().numpy()
    sel = 0
    for h in range(hq):
        kh = kv_of(h, hq, hkv)
        r = oracle.pbs_attention(q[h], k[kh], v[kh], ocfg(block_size=b, segment_size=s, tau=tau, strategy=strategy))
        np.testing.assert_array_equal(sigma[h], r.sigma)
        np.testing.assert_array_equal(pi[h], r.pi)
        np.testing.assert_array_equal(mask[h], r.mask)
        err = np.abs(out[h] - r.output)
        assert_bf16(err, h)
        sel += r.report["selected_blocks"]
    assert res.report["selected_blocks"] == sel


@pytest.mark.parametrize("strategy", ["key_permute", "none", "query_permute", "both"])
@pytest.mark.parametrize("n,b", [(1, 128), (100, 128), (128, 128), (129, 128), (383, 128),
                                 (1, 64), (63, 64), (65, 64), (129, 64), (300, 64)])
def test_pipeline_tiny_and_ragged_lengths(ops, oracle, monkeypatch, strategy, n, b):
    """Sequence lengths at and around one block on the tcgen05 path (d = 128,
    bf16, B = 128 and 64): a single key, a partial only block, exactly one
    block, one key past it, a segment plus a ragged block; at B = 64 also a
    lone query block in its tile pair."""
    from oracle import make_config as ocfg

    monkeypatch.setenv("PBS_REQUIRE_TC", "1")
    rng = np.random.default_rng(n)
    hq, hkv, d, s, tau = 2, 1, 128, 256, 0.9
    tq, tk, tv, q, k, v = bf16_inputs(rng, hq, hkv, n, d, kind="vertical_lines", strength=20.0)
    if strategy == "none":
        s = 0
    res = ops.pbs_attention(tq, tk, tv, ops.make_config(block_size=b, segment_size=s, tau=tau, strategy=strategy))
    out = res.output.float().cpu().numpy()
    assert np.isfinite(out).all()
    for h in range(hq):
        r = oracle.pbs_attention(q[h], k[0], v[0], ocfg(block_size=b, segment_size=s, tau=tau, strategy=strategy))
        np.testing.assert_array_equal(res.pi[h].cpu().numpy(), r.pi)
        np.testing.assert_array_equal(res.sigma[h].cpu().numpy(), r.sigma)
        np.testing.assert_array_equal(res.mask[h].cpu().numpy(), r.mask)
        err = np.abs(out[h] - r.output)
        assert_bf16(err, h)


@pytest.mark.parametrize("d,dtype", [(128, torch.bfloat16), (64, torch.float32), (20, torch.bfloat16)])
def test_unpermute_inverts_the_gather(ops, d, dtype):
    """pbs_unpermute (pipeline.hpp:178-180): out[sigma[i]] = src[i] == apply_rows(sigma^-1, src)."""
    g = torch.Generator(device="cuda").manual_seed(3)
    h, n = 3, 1000
    sigma = torch.stack([torch.randperm(n, generator=g, device="cuda") for _ in range(h)]).int()
    x = torch.randn(h, n, d, generator=g, device="cuda").to(dtype)
    xp = ops.apply_rows(sigma, x)
    assert torch.equal(ops.unpermute(sigma, xp), x)
    y = torch.randn(h, n, d, generator=g, device="cuda").to(dtype)
    got = ops.unpermute(sigma, y).float().cpu().numpy()
    for hh in range(h):
        inv = np.argsort(sigma[hh].cpu().numpy())  # Permutation::inverse (permutation.hpp:51-55)
        want = y[hh].float().cpu().numpy()[inv]   # apply_rows: out.row(i) = m.row(p[i]) (79-89)
        np.testing.assert_array_equal(got[hh], want)


@pytest.mark.parametrize("hq,hkv,n,b,kind", [(4, 2, 16384, 128, "vertical_lines"), (2, 1, 4096, 64, "gaussian"),
                                               (2, 2, 3000, 128, "adversarial")])
def test_query_permutation_screen_matches_exact(ops, oracle, monkeypatch, hq, hkv, n, b, kind):
    """build_query_permutation (permutation.hpp:206-275), bf16 d = 128: the
    tensor-core cosine screen + exact re-check equals the all-exact SIMT path and
    (sampled heads) the C restatement, including exact ties (duplicated key
    blocks -> identical centroids: smallest index), a zero-norm centroid, zero
    and anti-aligned queries."""
    rng = np.random.default_rng(21)
    d, seg = 128, 2 * b
    tq, tk, tv, q, k, v = bf16_inputs(rng, hq, hkv, n, d, kind="gaussian" if kind == "adversarial" else kind)
    if kind == "adversarial":
        k[:, 3 * b:4 * b] = k[:, 0:b]          # identical centroids 0 and 3
        k[:, 5 * b:6 * b] = k[:, 0:b]          # and 5
        k[:, 7 * b:8 * b] = 0.0                # zero-norm centroid
        cen = k[0, 0:b].mean(axis=0)
        q[:, 10:20] = cen * 4                   # exactly aligned with the tied centroids
        q[:, 20:30] = 0.0                       # zero-norm queries
        q[:, 30:40] = -cen                      # anti-aligned
        tq = torch.from_numpy(q).to(torch.bfloat16).cuda()
        tk = torch.from_numpy(k).to(torch.bfloat16).cuda()
        q, k = tq.float().cpu().numpy(), tk.float().cpu().numpy()
    perm_s, inv_s = ops.build_query_permutation(tq, tk, b, seg)
    monkeypatch.setenv("PBS_QGROUP_EXACT", "1")
    perm_e, inv_e = ops.build_query_permutation(tq, tk, b, seg)
    assert torch.equal(perm_s, perm_e) and torch.equal(inv_s, inv_e)
    for h in (0, hq - 1):
        want = oracle.build_query_permutation(q[h], k[kv_of(h, hq, hkv)], b, seg)
        np.testing.assert_array_equal(perm_s[h].cpu().numpy(), want)


@pytest.mark.parametrize("t,s_blocks,tau", [(256, 2, 0.9), (1024, 2, 0.9), (2048, 4, 0.75), (300, 1, 0.5)])
def test_select_exact_sum_path_edge_rows(ops, oracle, t, s_blocks, tau):
    """block_selection.hpp:171-206 on constructed rows: the order-free exact
    double-sum path (all candidates >= 2^-29) against the reference's sorted
    sequential sum, including ties at the tau boundary (broken by index), rows
    of equal probabilities, rows with tiny probabilities (< 2^-29: the sorted
    fallback) and unnormalised scores summing past 2 (fallback)."""
    rng = np.random.default_rng(11)
    b, seg = 64, 64 * s_blocks
    rows = []
    for i in range(t):
        kind = i % 6
        if kind == 0:
            r = rng.random(t).astype(np.float32)
        elif kind == 1:
            r = np.full(t, 1.0, np.float32)  # all ties
        elif kind == 2:
            r = np.round(rng.random(t) * 4).astype(np.float32)  # many ties on few levels
        elif kind == 3:
            r = (rng.random(t) * 1e-12).astype(np.float32)
            r[rng.integers(0, t, 3)] = 1.0  # a few large values, the rest below 2^-29
        elif kind == 4:
            r = rng.exponential(size=t).astype(np.float32) ** 4
        else:
            r = rng.random(t).astype(np.float32) * 8.0  # not normalised below
        rows.append(r)
    sc = np.stack(rows)
    causal = oracle.build_block_causal_mask(t, b, seg)
    # probabilities over each row's admissible prefix, as the pooled softmax produces
    adm = causal.astype(bool)
    p = np.where(adm, sc, 0).astype(np.float32)
    norm = p.sum(axis=1, keepdims=True).astype(np.float32)
    p = np.where(np.arange(t)[:, None] % 6 == 5, p, p / np.maximum(norm, 1e-30)).astype(np.float32)
    mask, kv_idx, kv_cnt = ops.select_blocks(torch.from_numpy(p[None]).cuda(), b, seg, tau)
    mask = mask.cpu().numpy()[0]
    wm = oracle.select_blocks(p, causal, b, seg, tau)
    np.testing.assert_array_equal(mask, wm)
    kv_cnt = kv_cnt.cpu().numpy()[0]
    np.testing.assert_array_equal(kv_cnt, wm.sum(axis=1))


@pytest.mark.parametrize("n,b,s,k", [(2048, 128, 256, 3), (4096, 16, 64, 40), (1000, 32, 64, 1)])
def test_select_top_k_bitexact(ops, oracle, n, b, s, k):
    """The top-k extension (north star (3)): the first k admissible blocks of the
    reference's stable order + forced blocks, against the C restatement."""
    rng = np.random.default_rng(8)
    tq, tk, tv, q, kk, v = bf16_inputs(rng, 2, 1, n, 64, kind="vertical_lines")
    scores = ops.meanpool_block_scores(tq, tk, b, s)
    mask, kv_idx, kv_cnt = ops.select_blocks(scores, b, s, 0.9, top_k=k)
    mask, kv_idx, kv_cnt, scores = mask.cpu().numpy(), kv_idx.cpu().numpy(), kv_cnt.cpu().numpy(), scores.cpu().numpy()
    t = -(-n // b)
    causal = oracle.build_block_causal_mask(t, b, s)
    for h in range(2):
        wm = oracle.select_blocks(scores[h], causal, b, s, 0.9, top_k=k)
        np.testing.assert_array_equal(mask[h], wm)
        for i in range(t):
            sel = np.flatnonzero(wm[i])
            assert kv_cnt[h, i] == sel.size
            np.testing.assert_array_equal(kv_idx[h, i, :sel.size], sel)


@pytest.mark.parametrize("k", [4, 32])
def test_pipeline_top_k_matches_oracle(ops, oracle, k):
    from oracle import make_config as ocfg

    rng = np.random.default_rng(12)
    hq, hkv, n, d, b, s = 2, 1, 4096, 128, 128, 256
    tq, tk, tv, q, kk, v = bf16_inputs(rng, hq, hkv, n, d, kind="vertical_lines", strength=20.0, block=b)
    res = ops.pbs_attention(tq, tk, tv, ops.make_config(block_size=b, segment_size=s, top_k=k))
    out, pi, mask = res.output.float().cpu().numpy(), res.pi.cpu().numpy(), res.mask.cpu().numpy()
    for h in range(hq):
        r = oracle.pbs_attention(q[h], kk[0], v[0], ocfg(block_size=b, segment_size=s, top_k=k))
        np.testing.assert_array_equal(pi[h], r.pi)
        np.testing.assert_array_equal(mask[h], r.mask)
        err = np.abs(out[h] - r.output)
        assert_bf16(err, h)
        # at most k + forced (block 0 and the row's segment band) per row
        assert (mask[h].sum(1) <= k + 1 + s // b).all()


@pytest.mark.parametrize("tau,top_k", [(0.0, 0), (0.9, 1000), (0.9, 1)])
@pytest.mark.parametrize("b", [128, 64])
def test_selection_extremes_match_oracle(ops, oracle, monkeypatch, tau, top_k, b):
    """tau = 0 (forced blocks only), top_k beyond every row's admissible count
    (everything admissible) and top_k = 1, through the whole pipeline, on the
    tensor-core path at B = 128 and B = 64."""
    from oracle import make_config as ocfg

    monkeypatch.setenv("PBS_REQUIRE_TC", "1")
    rng = np.random.default_rng(13)
    hq, hkv, n, d, s = 2, 1, 2048 + 77, 128, 256
    tq, tk, tv, q, kk, v = bf16_inputs(rng, hq, hkv, n, d, kind="vertical_lines", strength=20.0, block=b)
    res = ops.pbs_attention(tq, tk, tv, ops.make_config(block_size=b, segment_size=s, tau=tau, top_k=top_k))
    out, pi, mask = res.output.float().cpu().numpy(), res.pi.cpu().numpy(), res.mask.cpu().numpy()
    for h in range(hq):
        r = oracle.pbs_attention(q[h], kk[0], v[0], ocfg(block_size=b, segment_size=s, tau=tau, top_k=top_k))
        np.testing.assert_array_equal(pi[h], r.pi)
        np.testing.assert_array_equal(mask[h], r.mask)
        err = np.abs(out[h] - r.output)
        assert_bf16(err, h)
    if top_k >= 1000:
        assert res.report["selected_blocks"] == res.report["total_admissible_blocks"]


@pytest.mark.parametrize("kind", ["vertical_lines", "mixed", "gaussian"])
def test_reference_fixtures_f32(ops, kind):
    """The committed reference runs (oracle/gen_golden.py) through the f32 device path."""
    g = np.load(os.path.join(GOLDEN, f"ref_pipeline_f32_{kind}.npz"))
    meta = json.load(open(os.path.join(GOLDEN, "ref_pipeline_f32.json")))[kind]
    cfg = ops.make_config(block_size=meta["block"], segment_size=meta["segment"], tau=meta["tau"],
                          strategy=meta["strategy"])
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a[None])).cuda()  # noqa: E731
    res = ops.pbs_attention(t(g["q"]), t(g["k"]), t(g["v"]), cfg)
    np.testing.assert_array_equal(res.sigma.cpu().numpy()[0], g["sigma"])
    np.testing.assert_array_equal(res.pi.cpu().numpy()[0], g["pi"])
    np.testing.assert_array_equal(res.mask.cpu().numpy()[0], g["mask"])
    assert_f32(np.abs(res.output.cpu().numpy()[0] - g["output"]))
    for key in ("selected_blocks", "total_admissible_blocks"):
        assert res.report[key] == meta["report"][key]
    assert res.report["block_density"] == meta["report"]["block_density"]
    assert abs(res.report["pooled_score_coverage"] - meta["report"]["pooled_score_coverage"]) <= 1e-9


def test_causality_bitwise_on_device(ops):
    """pipeline_test.cpp:105-128 / acceptance C5 on the device path."""
    rng = np.random.default_rng(53)
    tq, tk, tv, *_ = bf16_inputs(rng, 2, 1, 1024, 128, kind="vertical_lines")
    cfg = ops.make_config(block_size=128, segment_size=256, tau=0.8)
    base = ops.pbs_attention(tq, tk, tv, cfg).output.clone()
    for j in (5, 300, 1023):
        v2 = tv.clone()
        v2[:, j] += 100.0
        out = ops.pbs_attention(tq, tk, v2, cfg).output
        assert torch.equal(out[:, :j], base[:, :j]), j


def test_dense_causal_matches_sdpa(ops):
    rng = np.random.default_rng(3)
    tq, tk, tv, *_ = bf16_inputs(rng, 8, 2, 2048 + 77, 128)
    out = ops.dense_causal_attention(tq, tk, tv).float()
    kk = tk.float().repeat_interleave(4, dim=0)
    vv = tv.float().repeat_interleave(4, dim=0)
    ref = torch.nn.functional.scaled_dot_product_attention(tq.float()[None], kk[None], vv[None], is_causal=True)[0]
    err = (out - ref).abs()
    assert_bf16(err)


@pytest.mark.parametrize("growth", [6.0, 40.0])
def test_dense_causal_running_max_growth(ops, growth):
    """Logits that grow along the keys (key norms ramp up), so the online
    softmax's running max rises block after block: the lazy rescale of O (max
    grows by more than 2^8) runs many times per row, in both softmax groups."""
    g = torch.Generator(device="cuda").manual_seed(5)
    n, d = 4096, 128
    q = torch.randn(2, n, d, device="cuda", generator=g)
    u = torch.randn(d, device="cuda", generator=g)
    q = (q + 2.0 * u).to(torch.bfloat16)
    ramp = torch.linspace(0.0, growth, n, device="cuda")[:, None]
    k = (torch.randn(1, n, d, device="cuda", generator=g) * 0.5 + ramp * u / u.norm()).to(torch.bfloat16)
    v = torch.randn(1, n, d, device="cuda", generator=g).to(torch.bfloat16)
    out = ops.dense_causal_attention(q, k, v).float()
    ref = torch.nn.functional.scaled_dot_product_attention(q.float()[None], k.float().expand(2, n, d)[None],
                                                           v.float().expand(2, n, d)[None], is_causal=True)[0]
    err = (out - ref).abs()
    assert_bf16(err)


def test_tau_one_is_causal_attention(ops):
    """pipeline_test.cpp:27-58 (C4) on device: tau = 1 selects the full causal grid."""
    rng = np.random.default_rng(5)
    tq, tk, tv, *_ = bf16_inputs(rng, 4, 2, 1024 + 128, 128)
    res = ops.pbs_attention(tq, tk, tv, ops.make_config(tau=1.0))
    dense = ops.dense_causal_attention(tq, tk, tv)
    err = (res.output.float() - dense.float()).abs()
    assert err.max().item() <= BF16_MAX


def test_degenerate_row_raises(ops):
    from paper_2510_21270_b200 import DegenerateRowError

    rng = np.random.default_rng(6)
    tq, tk, tv, *_ = bf16_inputs(rng, 1, 1, 512, 128)
    t = 4
    kv_idx = torch.zeros(1, t, t, dtype=torch.int32).cuda()
    kv_cnt = torch.tensor([[1, 0, 1, 1]], dtype=torch.int32).cuda()
    kv_idx[0, :, 0] = 0
    with pytest.raises(DegenerateRowError) as e:
        ops.attention_block_sparse(tq, tk, tv, 128, kv_idx, kv_cnt)
    assert "query block 1" in str(e.value)


# hkv = 1: one group; key_permute with hkv > 1: the estimate of every head runs
# up front (K streamed per KV head) and the groups take pi; query_permute with
# hkv > 1: per-group pipelines on two slots
@pytest.mark.parametrize("hq,hkv,n,strategy,b", [(2, 1, 1024, "key_permute", 128),
                                                 (8, 4, 2048 + 128, "key_permute", 128),
                                                 (6, 3, 1024, "query_permute", 128),
                                                 (8, 4, 2048 + 64 + 5, "key_permute", 64),
                                                 (6, 2, 1536, "both", 64)])
def test_host_entry_matches_device_entry(ops, hq, hkv, n, strategy, b):
    rng = np.random.default_rng(9)
    tq, tk, tv, *_ = bf16_inputs(rng, hq, hkv, n, 128, kind="vertical_lines")
    cfg = ops.make_config(strategy=strategy, block_size=b)
    dev = ops.pbs_attention(tq, tk, tv, cfg)
    host = ops.pbs_attention_host(tq.cpu(), tk.cpu(), tv.cpu(), cfg, return_perms=True)
    assert torch.equal(host.output, dev.output.cpu())
    assert torch.equal(host.pi, dev.pi.cpu())
    assert torch.equal(host.sigma, dev.sigma.cpu())
    assert torch.equal(host.mask, dev.mask.cpu())
    for key in ("selected_blocks", "total_admissible_blocks"):
        assert host.report[key] == dev.report[key]
    for key in ("block_density", "causal_density_baseline", "pooled_score_coverage"):
        assert abs(host.report[key] - dev.report[key]) < 1e-12


def test_cpp_dropin_runs(ops, tmp_path):
    """The C++ drop-in (examples/cpp_dropin.cpp) on the reference's configs[0] shape."""
    import subprocess

    from conftest import ROOT

    exe = tmp_path / "cpp_dropin"
    pkg = os.path.join(ROOT, "paper_2510_21270_b200")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "cpp_dropin.cpp"), "-L", pkg, "-lpbs_b200",
                    f"-Wl,-rpath,{pkg}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe), "4096", "128"], capture_output=True, text=True, check=True)
    rep = json.loads(r.stdout)
    assert 0 < rep["block_density"] <= rep["causal_density_baseline"] + 1e-9


def _torch_block_sparse_ref(q, k, v, b, kv_idx, kv_cnt, q_orig, k_orig, out_rows, scale):
    """attention_block_sparse (attention.hpp:259-310) restated densely in torch fp32:
    selected blocks AND the element mask k_orig[j] <= q_orig[i], then the row scatter."""
    hq, n, d = q.shape
    g = hq // k.shape[0]
    t = -(-n // b)
    out = torch.empty(hq, n, d, dtype=torch.float32, device=q.device)
    for h in range(hq):
        blk = torch.zeros(t, t, dtype=torch.bool, device=q.device)
        for i in range(t):
            c = int(kv_cnt[h, i])
            blk[i, kv_idx[h, i, :c].long()] = True
        sel = blk.repeat_interleave(b, 0).repeat_interleave(b, 1)[:n, :n]
        adm = k_orig[h][None, :] <= q_orig[h][:, None]
        s = (q[h].float() @ k[h // g].float().T) * scale
        s = s.masked_fill(~(sel & adm), float("-inf"))
        o = torch.softmax(s, dim=1) @ v[h // g].float()
        out[h, out_rows[h].long()] = o
    return out


@pytest.mark.parametrize("n,b", [(4096 + 50, 128), (6144, 128), (4096 + 50, 64), (3000, 64)])
def test_block_sparse_many_items_per_slot(ops, monkeypatch, n, b):
    """Several (head, query block) items per tensor-core slot (32 heads x 33-48
    blocks over 148 x 2 slots): Q reloads, O hand-over between items, K/V ring
    wrap-around, ragged final blocks, permuted original positions and the fused
    un-permute, against a dense torch restatement.  B = 64: every 128 x 128 tile
    carries four blocks selected (and classed) independently."""
    monkeypatch.setenv("PBS_REQUIRE_TC", "1")
    torch.manual_seed(0)
    hq, hkv, d, seg = 32, 8, 128, 256
    t = -(-n // b)
    q = torch.randn(hq, n, d, device="cuda").to(torch.bfloat16)
    k = torch.randn(hkv, n, d, device="cuda").to(torch.bfloat16)
    v = torch.randn(hkv, n, d, device="cuda").to(torch.bfloat16)
    # pi: a random permutation inside every segment (build_key_permutation's shape); sigma random too
    def seg_perm():
        p = torch.arange(n, device="cuda")
        for s0 in range(0, n - n % seg, seg):
            p[s0:s0 + seg] = s0 + torch.randperm(seg, device="cuda")
        return p
    k_orig = torch.stack([seg_perm() for _ in range(hq)]).int()
    q_orig = torch.stack([seg_perm() for _ in range(hq)]).int()
    # lists: block 0 + the segment band (the forced policy) + a random admissible subset, ascending
    kv_idx = torch.zeros(hq, t, t, dtype=torch.int32)
    kv_cnt = torch.zeros(hq, t, dtype=torch.int32)
    g = torch.Generator().manual_seed(1)
    per = seg // b
    for h in range(hq):
        for i in range(t):
            end = min((i // per + 1) * per, t)
            keep = torch.rand(end, generator=g) < 0.4
            keep[0] = True
            keep[(i // per) * per:end] = True
            sel = torch.nonzero(keep).flatten().int()
            kv_idx[h, i, :sel.numel()] = sel
            kv_cnt[h, i] = sel.numel()
    kv_idx, kv_cnt = kv_idx.cuda(), kv_cnt.cuda()
    out = ops.attention_block_sparse(q, k, v, b, kv_idx, kv_cnt, q_orig=q_orig, k_orig=k_orig, out_rows=q_orig)
    ref = _torch_block_sparse_ref(q, k, v, b, kv_idx, kv_cnt, q_orig, k_orig, q_orig, d ** -0.5)
    err = (out.float() - ref).abs()
    assert_bf16(err)


def test_dense_causal_many_items_per_slot(ops):
    """The dense comparator over 32 heads x 129 query blocks (~14 items per slot)
    against torch's own bf16 causal SDPA."""
    torch.manual_seed(2)
    hq, hkv, n, d = 32, 8, 16384 + 77, 128
    q = torch.randn(hq, n, d, device="cuda").to(torch.bfloat16)
    k = torch.randn(hkv, n, d, device="cuda").to(torch.bfloat16)
    v = torch.randn(hkv, n, d, device="cuda").to(torch.bfloat16)
    out = ops.dense_causal_attention(q, k, v)
    ref = torch.nn.functional.scaled_dot_product_attention(
        q[None], k.repeat_interleave(4, 0)[None], v.repeat_interleave(4, 0)[None], is_causal=True)[0]
    err = (out.float() - ref.float()).abs()
    assert_bf16(err)


@pytest.mark.parametrize("dtype,tol", [("f32", 1e-5), ("bf16", 1e-3)])
@pytest.mark.parametrize("strategy", ["key_permute", "query_permute", "none"])
def test_attention_coverage_matches_reference(ops, strategy, dtype, tol):
    """attention_coverage (pipeline.hpp:198-243) on the device (two attention
    passes, exp(lse_selected - lse_causal) per row) against the compiled
    reference on the same mask / sigma / pi.  f32 runs the CUDA-core kernel,
    bf16 the tcgen05 kernel (approximate exp2: 1e-3)."""
    import oracle as orc

    ref = orc.Oracle("ref") if orc.Oracle.available("ref") else orc.Oracle("oracle")
    rng = np.random.default_rng(23)
    hq, hkv, n, d, b, s = 2, 1, 1024 + 64, 128, 128, 256
    tq, tk, tv, q, k, v = bf16_inputs(rng, hq, hkv, n, d, kind="vertical_lines", strength=20.0)
    if dtype == "f32":
        tq, tk, tv = tq.float(), tk.float(), tv.float()
    cfg = ops.make_config(block_size=b, segment_size=0 if strategy == "none" else s, tau=0.8, strategy=strategy)
    res = ops.pbs_attention(tq, tk, tv, cfg)
    cov = ops.attention_coverage(tq, tk, res.mask, res.sigma, res.pi, b).numpy()
    sigma, pi, mask = res.sigma.cpu().numpy(), res.pi.cpu().numpy(), res.mask.cpu().numpy()
    for h in range(hq):
        want = ref.attention_coverage(q[h], k[kv_of(h, hq, hkv)], mask[h], b, sigma[h], pi[h])
        assert abs(cov[h] - want) <= tol, (h, cov[h], want)


def test_density_sweep_rows(ops):
    """density_sweep (pipeline.hpp:245-295): rows sorted by (segment, tau),
    density and coverage monotone in tau, tau = 1 exact against dense causal."""
    rng = np.random.default_rng(29)
    tq, tk, tv, *_ = bf16_inputs(rng, 4, 2, 2048, 128, kind="vertical_lines", strength=20.0)
    rows = ops.density_sweep(tq, tk, tv, ops.make_config(), [1.0, 0.5, 0.9], [512, 256])
    assert [(r.segment_size, r.tau) for r in rows] == [(256, 0.5), (256, 0.9), (256, 1.0), (512, 0.5),
                                                      (512, 0.9), (512, 1.0)]
    for a, c in zip(rows[:2], rows[1:3]):
        assert a.density <= c.density and a.coverage <= c.coverage + 1e-6
    full = rows[2]
    assert abs(full.coverage - 1.0) <= 1e-3 and full.max_err <= BF16_MAX
    assert all(r.time_us > 0 for r in rows)


def test_pipeline_cuda_graph_replay(ops):
    """The device pipeline (report=False, caller workspace) is stream-ordered and
    allocation-free, so the whole of Algorithm 1 (~20 launches) captures into
    one CUDA graph; replays reproduce the eager output bit for bit, also after
    the inputs are overwritten in place (the serving pattern)."""
    rng = np.random.default_rng(31)
    tq, tk, tv, *_ = bf16_inputs(rng, 8, 2, 4096, 128, kind="vertical_lines", strength=20.0)
    cfg = ops.make_config()
    ws = torch.empty(ops.workspace_size(tq, tk, cfg), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(tq)
    eager = ops.pbs_attention(tq, tk, tv, cfg, report=False, out=out, return_perms=False, ws=ws).output.clone()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):  # warm-up on the capture stream (one-time attribute setup)
        ops.pbs_attention(tq, tk, tv, cfg, report=False, out=out, return_perms=False, ws=ws)
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ops.pbs_attention(tq, tk, tv, cfg, report=False, out=out, return_perms=False, ws=ws)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)
    tq2, tk2, tv2, *_ = bf16_inputs(np.random.default_rng(32), 8, 2, 4096, 128, kind="vertical_lines")
    want = ops.pbs_attention(tq2, tk2, tv2, cfg).output
    tq.copy_(tq2), tk.copy_(tk2), tv.copy_(tv2)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, want)


def test_pipeline_qwen_gqa_group_of_seven(ops, oracle):
    """Qwen2.5-7B's GQA (28 q / 4 kv heads: groups of 7, BASELINE configs[3]) on
    one group plus a 3 + 4 split of it (the 8-GPU shard shape): permutations and
    masks bit-exact, outputs to the bf16 tolerance."""
    from oracle import make_config as ocfg

    rng = np.random.default_rng(37)
    tq, tk, tv, q, k, v = bf16_inputs(rng, 7, 1, 2048 + 64, 128, kind="vertical_lines", strength=20.0)
    cfg = ops.make_config(tau=0.9)
    full = ops.pbs_attention(tq, tk, tv, cfg)
    for lo, hi in ((0, 3), (3, 7)):
        part = ops.pbs_attention(tq[lo:hi].contiguous(), tk, tv, cfg)
        assert torch.equal(part.output, full.output[lo:hi])
        assert torch.equal(part.mask, full.mask[lo:hi])
    for h in range(7):
        r = oracle.pbs_attention(q[h], k[0], v[0], ocfg(block_size=128, segment_size=256, tau=0.9))
        np.testing.assert_array_equal(full.pi[h].cpu().numpy(), r.pi)
        np.testing.assert_array_equal(full.mask[h].cpu().numpy(), r.mask)
        err = np.abs(full.output[h].float().cpu().numpy() - r.output)
        assert_bf16(err)


@pytest.mark.parametrize("d", [192, 256])
def test_simt_attention_large_head_dims(ops, oracle, d):
    """Head dims 192 / 256 on the CUDA-core attention (more than the 48 KB
    default of dynamic shared memory), through the whole pipeline."""
    from oracle import make_config as ocfg

    rng = np.random.default_rng(d)
    hq, hkv, n, b, s = 2, 1, 640, 64, 128
    tq, tk, tv, q, k, v = bf16_inputs(rng, hq, hkv, n, d, kind="vertical_lines", strength=20.0, block=b)
    res = ops.pbs_attention(tq, tk, tv, ops.make_config(block_size=b, segment_size=s, tau=0.9))
    out = res.output.float().cpu().numpy()
    for h in range(hq):
        r = oracle.pbs_attention(q[h], k[0], v[0], ocfg(block_size=b, segment_size=s, tau=0.9))
        np.testing.assert_array_equal(res.pi[h].cpu().numpy(), r.pi)
        np.testing.assert_array_equal(res.mask[h].cpu().numpy(), r.mask)
        assert_bf16(np.abs(out[h] - r.output), h)


@pytest.mark.parametrize("segment", [4096 + 7, 8192])
def test_key_permutation_large_segments(ops, oracle, segment):
    """Segments of 4097..8192 keys (64 KB of shared memory in the device sort)."""
    rng = np.random.default_rng(segment)
    n = 2 * segment + 100
    scores = rng.standard_normal((2, n)).astype(np.float32)
    scores[:, ::5] = 0.25  # ties
    perm, inv = ops.build_key_permutation(torch.from_numpy(scores).cuda(), segment)
    perm = perm.cpu().numpy()
    for h in range(2):
        np.testing.assert_array_equal(perm[h], oracle.build_key_permutation(scores[h], segment))
        np.testing.assert_array_equal(inv.cpu().numpy()[h][perm[h]], np.arange(n))


def test_host_entry_concurrent_callers(ops):
    """Two host threads calling the host-buffer entry at once (each checks out
    its own arena): both results equal their single-caller runs."""
    import threading

    rng = np.random.default_rng(21)
    cfg = ops.make_config()
    probs = []
    for _ in range(2):
        tq, tk, tv, *_ = bf16_inputs(rng, 8, 2, 2048, 128, kind="vertical_lines")
        probs.append((tq.cpu(), tk.cpu(), tv.cpu()))
    want = [ops.pbs_attention_host(*p, cfg, return_perms=True) for p in probs]
    got = [None, None]
    errs = []

    def run(i):
        try:
            for _ in range(3):
                got[i] = ops.pbs_attention_host(*probs[i], cfg, return_perms=True)
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)

    ths = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errs, errs
    for w, g in zip(want, got):
        assert torch.equal(w.output, g.output) and torch.equal(w.pi, g.pi) and torch.equal(w.mask, g.mask)
        assert w.report["selected_blocks"] == g.report["selected_blocks"]


# ---- head-parallel shards on the device -------------------
@pytest.mark.parametrize("hq,hkv,n,world,b", [(8, 2, 2048, 2, 128), (8, 2, 2048 + 64, 4, 128),
                                              (14, 2, 4096, 4, 128), (7, 1, 2048, 2, 128),
                                              (7, 1, 4096 + 128, 8, 128), (3, 3, 640, 8, 128),
                                              (7, 1, 4096 + 64 + 9, 4, 64), (8, 2, 3072, 8, 64)])
def test_shards_reassemble_pbs_attention(ops, hq, hkv, n, world, b):
    """Every rank's pbs_attention_shard run one after another on this GPU into
    one buffer equals the single pbs_attention call bit for bit -- including
    ranks whose share cuts inside a head (Qwen-like groups of 7) and ranks
    that need only some KV heads; the reports sum to the single call's."""
    rng = np.random.default_rng(hq * n + world)
    tq, tk, tv, *_ = bf16_inputs(rng, hq, hkv, n, 128, kind="vertical_lines")
    cfg = ops.make_config(block_size=b)
    want = ops.pbs_attention(tq, tk, tv, cfg)
    out = torch.zeros_like(tq)
    sel = 0
    cuts = 0
    for r in range(world):
        s = ops.shard_plan(hq, hkv, n, 128, b, world, r)
        if s["out_rows"] == 0:
            continue
        cuts += s["qb_begin"] != 0
        ql = tq[s["head_begin"]:s["head_end"]].contiguous()
        kl = tk[s["kv_begin"]:s["kv_end"]].contiguous()
        vl = tv[s["kv_begin"]:s["kv_end"]].contiguous()
        rep = ops.attention_shard(ql, kl, vl, hq, hkv, cfg, world, r, out, report=True)
        sel += rep["selected_blocks"]
    torch.cuda.synchronize()
    assert torch.equal(out, want.output)
    assert sel == want.report["selected_blocks"]
    if hq % world:
        assert cuts > 0  # the split really cut inside a head


def test_dist_context_world_one_matches(ops):
    """pbs_dist_* with a one-rank NCCL communicator: compute + the (trivial)
    in-place broadcast equals pbs_attention; the global report matches."""
    rng = np.random.default_rng(31)
    tq, tk, tv, *_ = bf16_inputs(rng, 8, 2, 2048, 128, kind="vertical_lines")
    cfg = ops.make_config()
    want = ops.pbs_attention(tq, tk, tv, cfg)
    ctx = ops.DistContext(ops.dist_unique_id(), 1, 0)
    out = torch.zeros_like(tq)
    rep = ctx.attention(tq, tk, tv, 8, 2, cfg, out, report=True)
    torch.cuda.synchronize()
    ctx.close()
    assert torch.equal(out, want.output)
    for key in ("selected_blocks", "total_admissible_blocks"):
        assert rep[key] == want.report[key]
    assert abs(rep["block_density"] - want.report["block_density"]) < 1e-12


def _two_process_worker(rank, world, port, path):
    import torch.distributed as dist

    from paper_2510_21270_b200 import ops as o

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    rng = np.random.default_rng(77)
    hq, hkv, n = 7, 1, 2048
    tq, tk, tv, *_ = bf16_inputs(rng, hq, hkv, n, 128, kind="vertical_lines")
    cfg = o.make_config()
    s = o.shard_plan(hq, hkv, n, 128, 128, world, rank)
    out = torch.zeros_like(tq)
    o.attention_shard(tq[s["head_begin"]:s["head_end"]].contiguous(), tk[s["kv_begin"]:s["kv_end"]].contiguous(),
                      tv[s["kv_begin"]:s["kv_end"]].contiguous(), hq, hkv, cfg, world, rank, out)
    full = out.cpu().reshape(-1, 128)
    for r in range(world):  # the all-gather-v over gloo (the product does it with NCCL)
        sr = o.shard_plan(hq, hkv, n, 128, 128, world, r)
        view = full[sr["out_row_begin"]:sr["out_row_begin"] + sr["out_rows"]]
        buf = view.float().clone()
        dist.broadcast(buf, src=r)
        view.copy_(buf.to(view.dtype))
    if rank == 0:
        want = o.pbs_attention(tq, tk, tv, cfg).output.cpu().reshape(-1, 128)
        torch.save({"ok": bool(torch.equal(full, want))}, path)
    dist.barrier()
    dist.destroy_process_group()


def test_two_processes_one_gpu_gather(ops, tmp_path):
    """Two processes (gloo for the exchange) each run their shard of a
    Qwen-like group of 7 on the device pipeline; the gathered output equals
    the single-process result bit for bit."""
    import socket

    import torch.multiprocessing as mp

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    path = str(tmp_path / "ok.pt")
    mp.spawn(_two_process_worker, args=(2, port, path), nprocs=2, join=True)
    assert torch.load(path)["ok"]


# ---------------------------------------------------------------------------
def test_c1_config_end_to_end_matches_reference(ops, ref):
    """BASELINE configs[0] (C1): one head, N = 4096, d = 128, B = 64, S = 256,
    tau = 0.9, key_permute, fp32, inputs from the reference's own generator
    (pbs::generate_head, vertical lines, seed 1, 16 lines of strength 150;
    workload.hpp:145-198), run by the unmodified reference pbs_attention
    (pipeline.hpp:107-193) and by both device entries (inputs resident, and the
    host-buffer call).  pi / sigma / mask / counts bit-exact, output within the
    f32 bar (scripts/c1_bench.py times the same case)."""
    from oracle import make_config as ref_config
    from oracle.gen_golden import generate_head

    n, d, b, s, tau = 4096, 128, 64, 256, 0.9
    q, k, v, _ = generate_head(ref, "vertical_lines", n, d, 1, b, s, line_count=16, line_strength=150.0,
                               dtype=np.float32)
    rr = ref.pbs_attention(q, k, v, ref_config(block_size=b, segment_size=s, tau=tau, strategy="key_permute"))
    cfg = ops.make_config(block_size=b, segment_size=s, tau=tau, strategy="key_permute")
    tq, tk, tv = (torch.from_numpy(x[None].copy()) for x in (q, k, v))
    dev = ops.pbs_attention(tq.cuda(), tk.cuda(), tv.cuda(), cfg)
    host = ops.pbs_attention_host(tq, tk, tv, cfg, return_perms=True)
    for res in (dev, host):
        np.testing.assert_array_equal(res.pi.cpu().numpy()[0], rr.pi)
        np.testing.assert_array_equal(res.sigma.cpu().numpy()[0], rr.sigma)
        np.testing.assert_array_equal(res.mask.cpu().numpy()[0], rr.mask)
        assert_f32(np.abs(res.output.cpu().numpy()[0] - rr.output))
        for key in ("selected_blocks", "total_admissible_blocks"):
            assert res.report[key] == rr.report[key]
        assert res.report["block_density"] == rr.report["block_density"]
