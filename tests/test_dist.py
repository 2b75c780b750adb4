"""Multi-rank host logic of the head-parallel path, on CPU.

The product splits the work with pbs_shard_plan (csrc/dist.cu): contiguous
ranges of (query head, query-block pair) units holding equal causal work, so
each rank's output rows are one contiguous range of the [Hq * N] output and
the one exchange is an all-gather-v (one broadcast per rank).  Here:
  * the plan itself (coverage, contiguity, balance, KV ranges) for the bench
    shapes at 1/2/4/8 ranks, against a Python restatement of the work model;
  * 2 and 8 gloo ranks run that exact split on a small problem, compute their
    rows with the CPU oracle (standing in for the device pipeline, which
    tests/test_gpu_parity.py::test_shards_reassemble_* runs rank by rank) and
    exchange them with the same per-rank broadcasts; the result must equal the
    single-rank run bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_21270_b200 import ops

N_SMALL = 512
B_SMALL, S_SMALL = 64, 128


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _use_model(name):
    import bench

    bench.HQ, bench.HKV, bench.N, bench.PREFIX = bench.MODELS[name]
    return bench


def _per(b):
    """Query blocks per unit: a pair of 128-row tiles (4 blocks at B = 64), else 2."""
    return 4 if b == 64 else 2


def _pair_work(t, per=2):
    """Causal key blocks visited per (head, unit): query blocks per*p .. per*p + per - 1."""
    return [sum(qb + 1 for qb in range(per * p, min(per * p + per, t))) for p in range(-(-t // per))]


@pytest.mark.parametrize("hq,hkv,n,b", [(32, 8, 131072, 128), (28, 4, 262144, 128), (32, 8, 32768, 128),
                                        (28, 4, N_SMALL, B_SMALL), (6, 3, 1000, 64), (1, 1, 4096, 64),
                                        (5, 5, 129, 128)])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_plan_covers_balances_and_is_contiguous(hq, hkv, n, b, world):
    t = -(-n // b)
    per = _per(b)
    w = _pair_work(t, per)
    owner = {}
    rows = []
    loads = []
    for r in range(world):
        s = ops.shard_plan(hq, hkv, n, 128, b, world, r)
        load = 0
        for h in range(s["head_begin"], s["head_end"]):
            lo = s["qb_begin"] if h == s["head_begin"] else 0
            hi = s["qb_end"] if h == s["head_end"] - 1 else t
            assert lo % per == 0 and (hi % per == 0 or hi == t) and lo < hi
            for p in range(lo // per, -(-hi // per)):
                assert (h, p) not in owner
                owner[(h, p)] = r
                load += w[p]
        if s["out_rows"]:
            assert s["kv_begin"] == s["head_begin"] // (hq // hkv)
            assert s["kv_end"] == (s["head_end"] - 1) // (hq // hkv) + 1
            rows.append((s["out_row_begin"], s["out_rows"]))
        loads.append(load)
    assert len(owner) == hq * len(w)  # every unit exactly once
    start = 0
    for r0, cnt in rows:  # contiguous, in rank order, tiling [0, Hq * N)
        assert r0 == start
        start += cnt
    assert start == hq * n
    mean = sum(loads) / world
    assert max(loads) - mean <= max(w) + 1e-9  # balanced to one unit
    if hq % world == 0:  # whole heads when they split evenly
        for r in range(world):
            s = ops.shard_plan(hq, hkv, n, 128, b, world, r)
            assert s["qb_begin"] == 0 and s["qb_end"] == t and s["head_end"] - s["head_begin"] == hq // world


def test_qwen_on_8_ranks_is_balanced_not_4_plus_3():
    """28 heads on 8 ranks: 3.5 heads of work each (the 4 + 3 head split caps
    efficiency at 87.5%)."""
    t = 262144 // 128
    w = _pair_work(t)
    head_w = sum(w)
    loads = []
    for r in range(8):
        s = ops.shard_plan(28, 4, 262144, 128, 128, 8, r)
        load = 0
        for h in range(s["head_begin"], s["head_end"]):
            lo = s["qb_begin"] if h == s["head_begin"] else 0
            hi = s["qb_end"] if h == s["head_end"] - 1 else t
            load += sum(w[lo // 2:-(-hi // 2)])
        loads.append(load / head_w)
    assert max(loads) - min(loads) < 2 * max(w) / head_w
    assert abs(np.mean(loads) - 3.5) < 1e-9


def _oracle_rows(model, world, rank):
    """The rank's rows of the [Hq, N, d] output from the CPU oracle (whole heads
    computed, the shard's rows kept), flattened [rows, d]."""
    import oracle

    bench = _use_model(model)
    s = ops.shard_plan(bench.HQ, bench.HKV, N_SMALL, 128, B_SMALL, world, rank)
    if s["out_rows"] == 0:
        return s, torch.zeros(0, 128)
    kv_list = list(range(s["kv_begin"], s["kv_end"]))
    q, k, v = bench.make_inputs(torch, N_SMALL, s["head_begin"], s["head_end"], kv_list, "cpu")
    orc = oracle.Oracle("oracle")
    cfg = oracle.make_config(block_size=B_SMALL, segment_size=S_SMALL, tau=0.9, strategy="key_permute")
    g = bench.HQ // bench.HKV
    outs = []
    for j, h in enumerate(range(s["head_begin"], s["head_end"])):
        kv = h // g - s["kv_begin"]
        r = orc.pbs_attention(q[j].float().numpy(), k[kv].float().numpy(), v[kv].float().numpy(), cfg)
        outs.append(torch.from_numpy(r.output))
    flat = torch.stack(outs).reshape(-1, 128)
    r0 = s["out_row_begin"] - s["head_begin"] * N_SMALL
    return s, flat[r0:r0 + s["out_rows"]]


def _worker(rank, world, port, path, model):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bench = _use_model(model)
    full = torch.zeros(bench.HQ * N_SMALL, 128)
    s, mine = _oracle_rows(model, world, rank)
    if s["out_rows"]:
        full[s["out_row_begin"]:s["out_row_begin"] + s["out_rows"]] = mine
    # the product's exchange: one broadcast of each rank's contiguous rows (all-gather-v)
    for r in range(world):
        sr = ops.shard_plan(bench.HQ, bench.HKV, N_SMALL, 128, B_SMALL, world, r)
        if sr["out_rows"]:
            view = full[sr["out_row_begin"]:sr["out_row_begin"] + sr["out_rows"]]
            buf = view.clone()
            dist.broadcast(buf, src=r)
            view.copy_(buf)
    if rank == world - 1:
        torch.save(full.reshape(bench.HQ, N_SMALL, 128), path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.fixture(autouse=True)
def _restore_bench_model():
    yield
    _use_model("llama")


@pytest.mark.parametrize("model,world", [("llama", 2), ("qwen", 2), ("qwen", 8)])
def test_multi_rank_gather_matches_single_rank(tmp_path, model, world):
    path = str(tmp_path / "gathered.pt")
    mp.spawn(_worker, args=(world, _free_port(), path, model), nprocs=world, join=True)
    gathered = torch.load(path)
    _, single = _oracle_rows(model, 1, 0)
    bench = _use_model(model)
    assert gathered.shape == (bench.HQ, N_SMALL, 128)
    assert torch.equal(gathered.reshape(-1, 128), single)
