"""Bit-exact parity at the bench's own configurations against the compiled
reference (oracle/_ref/libpbsref.so: the unmodified reference headers).

Configs (BASELINE.json configs[1..3]), inputs from
``bench.make_inputs`` -- the exact tensors the bench times:
  * C2  Llama-3.1-8B shapes (32 q / 8 kv heads, d = 128) at N = 32768;
  * C3  the same at N = 131072 (the headline);
  * C4  Qwen2.5-7B shapes (28 q / 4 kv heads) at N = 262144.
B = 128, S = 256, tau = 0.9, key_permute; C2 also at B = 64 (the
block-size variant, two selection blocks per tensor-core tile side).

For EVERY query head, on the bf16-upcast inputs (exact in f32):
  * importance scores (permutation.hpp:143-178) bit for bit;
  * pi (permutation.hpp:182-201) equal;
  * pooled block scores (block_selection.hpp:120-161) over Q and pi K bit for bit;
  * mask (block_selection.hpp:171-206) equal, and the pipeline's report count.
The reference runs one head per host thread (ctypes releases the GIL), like
pbs_main.cpp:99-122.  The tie audit SURVEY.md §8c asks for (adjacent sorted
pairs inside a segment with relative gap < 1e-6, exact ties separately) is
computed per config and written to $PBS_AUDIT_DIR when set.

Attention outputs at these sizes are checked on sampled rows against fp32
softmax over exactly the selected keys in tests/test_fullsize_properties.py.
"""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
S, TAU = 256, 0.9

CONFIGS = {"c2_llama_32k": ("llama", 32768, 128), "c3_llama_128k": ("llama", 131072, 128),
           "c4_qwen_256k": ("qwen", 262144, 128), "c2_llama_32k_b64": ("llama", 32768, 64)}


def _audit(sorted_scores):
    """Adjacent pairs inside each segment of the pi-sorted scores: exact ties and
    relative gaps below 1e-6 (non-zero)."""
    a, b = sorted_scores[:, :-1], sorted_scores[:, 1:]
    exact = int((a == b).sum())
    den = np.maximum(np.abs(a), np.abs(b))
    near = int(((a != b) & (np.abs(a - b) < 1e-6 * den)).sum())
    return exact, near


@pytest.fixture(scope="module", params=sorted(CONFIGS))
def fullsize(request):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from oracle import Oracle

    if not Oracle.available("ref"):
        pytest.skip("oracle/_ref/libpbsref.so not built")
    import bench
    from paper_2510_21270_b200 import ops

    model, n, B = CONFIGS[request.param]
    hq, hkv, _, prefix = bench.MODELS[model]
    bench.HQ, bench.HKV, bench.PREFIX = hq, hkv, prefix
    q, k, v = bench.make_inputs(torch, n, 0, hq, list(range(hkv)), "cuda")
    cfg = ops.make_config(block_size=B, segment_size=S, tau=TAU, strategy="key_permute")
    res = ops.pbs_attention(q, k, v, cfg, report=True, return_perms=True)
    scores = ops.estimate_key_importance(q, k, B)
    bscores = ops.meanpool_block_scores(q, ops.apply_rows(res.pi, k, hq), B, S)
    dev = {"scores": scores.cpu().numpy(), "pi": res.pi.cpu().numpy(), "mask": res.mask.cpu().numpy(),
           "bscores": bscores.cpu().numpy(), "report": res.report}
    qh = q.float().cpu().numpy()
    kh = k.float().cpu().numpy()
    del q, k, v, res, scores, bscores
    torch.cuda.empty_cache()
    yield request.param, hq, hkv, n, B, qh, kh, dev


def test_fullsize_pi_and_mask_equal_reference(fullsize):
    from oracle import Oracle

    name, hq, hkv, n, B, q, k, dev = fullsize
    ref = Oracle("ref")
    g = hq // hkv
    t = n // B
    causal = ref.build_block_causal_mask(t, B, S)

    def one(h):
        kk = k[h // g]
        sc, _ = ref.estimate_key_importance(q[h], kk, B)
        pi = ref.build_key_permutation(sc, S)
        bs = ref.meanpool_block_scores(q[h], kk[pi], B, causal)
        mask = ref.select_blocks(bs, causal, B, S, TAU)
        return {
            "scores": int(np.count_nonzero(sc.view(np.uint32) != dev["scores"][h].view(np.uint32))),
            "pi": int(np.count_nonzero(pi != dev["pi"][h])),
            "bscores": int(np.count_nonzero(bs.view(np.uint32) != dev["bscores"][h].view(np.uint32))),
            "mask": int(np.count_nonzero(mask != dev["mask"][h])),
            "selected": int(mask.sum()),
            "audit": _audit(sc[pi].reshape(-1, S)),
        }

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=min(hq, os.cpu_count() or 1)) as ex:
        rows = list(ex.map(one, range(hq)))
    wall = time.perf_counter() - t0
    bad = {h: r for h, r in enumerate(rows) if any(r[x] for x in ("scores", "pi", "bscores", "mask"))}
    summary = {
        "config": name, "q_heads": hq, "kv_heads": hkv, "seq_len": n, "block": B, "segment": S, "tau": TAU,
        "heads_checked": hq, "heads_mismatching": len(bad),
        "selected_blocks": sum(r["selected"] for r in rows),
        "device_selected_blocks": dev["report"]["selected_blocks"],
        "tie_audit": {"exact_ties": sum(r["audit"][0] for r in rows),
                      "near_ties_rel_lt_1e-6": sum(r["audit"][1] for r in rows),
                      "adjacent_pairs": hq * (n // S) * (S - 1)},
        "reference_cpu_s": round(wall, 2), "threads": min(hq, os.cpu_count() or 1),
    }
    out_dir = os.environ.get("PBS_AUDIT_DIR")
    if out_dir:
        os.makedirs(out_dir, exist_ok=True)
        with open(os.path.join(out_dir, f"parity_{name}.json"), "w") as f:
            json.dump({**summary, "mismatches": bad}, f, indent=1)
    print(json.dumps(summary))
    assert not bad, f"{len(bad)} heads differ from the reference: {dict(list(bad.items())[:4])}"
    assert summary["selected_blocks"] == summary["device_selected_blocks"]
