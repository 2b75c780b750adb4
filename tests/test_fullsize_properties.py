"""C3 and C4 at their full sizes (Llama-3.1-8B shapes, 32 q / 8 kv heads at
N = 131072; Qwen2.5-7B shapes, 28 q / 4 kv heads at N = 262144; bf16, B = 128,
S = 256, tau = 0.9): properties that hold at any size, checked where the CPU
oracle cannot follow.

  * pi: within every segment a permutation of the segment's own indices,
    ordering the importance scores non-increasingly (ties by index);
  * masks: nothing above the segment band, block 0 and the whole diagonal band
    present, the kv lists ascending and equal to the mask rows, the report's
    counts equal to the masks';
  * outputs: finite, and for sampled rows equal (bf16 tolerance) to softmax
    attention restricted to exactly the selected permuted key blocks and the
    causal element mask, computed directly in fp32;
  * tau = 1: every admissible block selected (density = the causal baseline).
"""
import os
import sys

import pytest

from conftest import assert_bf16

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
B, S = 128, 256


@pytest.fixture(scope="module", params=["llama", "qwen"])
def c3(request):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import bench
    from paper_2510_21270_b200 import ops
    hq, hkv, n, prefix = bench.MODELS[request.param]
    bench.HQ, bench.HKV, bench.N, bench.PREFIX = hq, hkv, n, prefix
    q, k, v = bench.make_inputs(torch, n, 0, hq, list(range(hkv)), "cuda")
    cfg = ops.make_config(block_size=B, segment_size=S, tau=0.9, strategy="key_permute")
    res = ops.pbs_attention(q, k, v, cfg, report=True, return_perms=True)
    yield ops, q, k, v, res
    del q, k, v, res
    torch.cuda.empty_cache()


def test_pi_is_a_sorted_segment_permutation(c3):
    ops, q, k, v, res = c3
    hq, N = q.shape[0], q.shape[1]
    pi = res.pi.long()
    seg = pi.view(hq, N // S, S)
    base = (torch.arange(N // S, device="cuda") * S)[None, :, None]
    assert torch.equal(seg.sort(dim=2).values - base, torch.arange(S, device="cuda").expand_as(seg))
    scores = ops.estimate_key_importance(q, k, B)
    sp = torch.gather(scores, 1, pi).view(hq, N // S, S)
    assert bool((sp[..., :-1] >= sp[..., 1:]).all())  # non-increasing inside every segment
    ties = sp[..., :-1] == sp[..., 1:]
    local = seg - base
    assert bool((local[..., :-1][ties] < local[..., 1:][ties]).all())  # ties keep ascending order


def test_masks_respect_band_and_forced_blocks(c3):
    ops, q, k, v, res = c3
    hq, N = q.shape[0], q.shape[1]
    t = N // B
    mask = res.mask.bool()
    i = torch.arange(t, device="cuda")
    seg = i // (S // B)
    above = seg[None, :] > seg[:, None]  # key block segment after the query block's
    assert not bool(mask[:, above].any())
    assert bool(mask[:, :, 0].all())
    band = seg[None, :] == seg[:, None]
    assert bool(mask[:, band].all())
    assert int(mask.sum()) == res.report["selected_blocks"]
    # the attention lists: same sets, ascending
    # key_permute: sigma = identity, so the pooled queries are Q's and the pooled keys K' = pi K's
    scores = ops.meanpool_block_scores(q, ops.apply_rows(res.pi, k, hq), B, S)
    m2, kv_idx, kv_cnt = ops.select_blocks(scores, B, S, 0.9)
    assert torch.equal(m2, res.mask)
    assert torch.equal(kv_cnt, mask.sum(2).int())
    for h in (0, 17, hq - 1):
        for r in (0, 1, 511, t - 1):
            c = int(kv_cnt[h, r])
            lst = kv_idx[h, r, :c]
            assert torch.equal(lst, torch.nonzero(mask[h, r]).flatten().int())


def test_sampled_rows_equal_restricted_softmax(c3):
    ops, q, k, v, res = c3
    hq, N = q.shape[0], q.shape[1]
    g = hq // k.shape[0]
    assert bool(torch.isfinite(res.output.float()).all())
    scale = 1.0 / 128 ** 0.5
    for h, i in [(0, 0), (0, 777), (5, 65535), (13, 100000), (hq - 1, N - 1), (20, N - 72)]:
        kv = h // g
        qb = i // B
        blocks = torch.nonzero(res.mask[h, qb]).flatten()
        keys = res.pi[h].view(-1, B)[blocks].flatten().long()  # original positions of the selected keys
        keys = keys[keys <= i]  # ElementMask: k_orig <= q_orig (sigma = identity)
        s = (q[h, i].float() @ k[kv, keys].float().T) * scale
        p = torch.softmax(s, dim=0)
        want = p @ v[kv, keys].float()
        got = res.output[h, i].float()
        assert_bf16((got - want).abs(), (h, i))


def test_tau_one_selects_every_admissible_block(c3):
    ops, q, k, v, res = c3
    r = ops.pbs_attention(q, k, v, ops.make_config(block_size=B, segment_size=S, tau=1.0), report=True,
                          return_perms=False).report
    assert r["selected_blocks"] == r["total_admissible_blocks"]
    assert abs(r["block_density"] - r["causal_density_baseline"]) < 1e-2
