"""Multi-rank host logic of the head-parallel path, on CPU.

bench.py shards query heads along KV groups and assembles the output with one
all-gather.  Here 2 gloo ranks run that exact sharding on a small problem,
compute each local head with the CPU oracle (standing in for the device
pipeline) and all-gather; the result must equal the single-rank run bit for
bit, i.e. the shard boundaries, per-KV-head seeding and gather order
reproduce the N = 1 problem.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N_SMALL = 512


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


def _local_outputs(rank, world, model="llama", pad_to=None):
    import oracle

    bench = _use_model(model)
    q0, q1, kv_list, g_local = bench.shard_of(rank, world)
    q, k, v = bench.make_inputs(torch, N_SMALL, q0, q1, kv_list, "cpu")
    orc = oracle.Oracle("oracle")
    cfg = oracle.make_config(block_size=64, segment_size=128, tau=0.9, strategy="key_permute")
    outs = []
    for h in range(q1 - q0):
        r = orc.pbs_attention(q[h].float().numpy(), k[h // g_local].float().numpy(), v[h // g_local].float().numpy(),
                              cfg)
        outs.append(torch.from_numpy(r.output))
    out = torch.stack(outs)
    if pad_to is not None and out.shape[0] < pad_to:  # bench.py pads the gather to the largest share
        out = torch.cat([out, torch.zeros(pad_to - out.shape[0], *out.shape[1:])])
    return out


def _worker(rank, world, port, path, model):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bench = _use_model(model)
    shares = [bench.shard_of(r, world) for r in range(world)]
    max_local = max(s[1] - s[0] for s in shares)
    out = _local_outputs(rank, world, model, pad_to=max_local)
    full = [torch.empty_like(out) for _ in range(world)]
    dist.all_gather(full, out)
    if rank == 0:  # drop each rank's padding, in rank order
        torch.save(torch.cat([f[:s[1] - s[0]] for f, s in zip(full, shares)]), path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("model", ["llama", "qwen"])
def test_shard_arithmetic(model):
    """Every query head owned exactly once; each local query head reads the KV
    head of its group; Llama splits whole groups, Qwen's groups of 7 split 3 + 4
    on 8 ranks with both halves holding the group's KV head."""
    bench = _use_model(model)
    g = bench.HQ // bench.HKV
    for world in (1, 2, 4, 8):
        owned = []
        for r in range(world):
            q0, q1, kv_list, g_local = bench.shard_of(r, world)
            assert (q1 - q0) == len(kv_list) * g_local
            for j, h in enumerate(range(q0, q1)):
                assert kv_list[j // g_local] == h // g
            owned += list(range(q0, q1))
        assert owned == list(range(bench.HQ))
    if model == "qwen":
        assert [bench.shard_of(r, 8)[1] - bench.shard_of(r, 8)[0] for r in range(8)] == [3, 4] * 4
    else:
        assert all(bench.shard_of(r, 8)[3] == 4 for r in range(8))
    with pytest.raises(ValueError):
        bench.shard_of(0, bench.HQ + 1)


@pytest.fixture(autouse=True)
def _restore_bench_model():
    yield
    _use_model("llama")


@pytest.mark.parametrize("model,world", [("llama", 2), ("qwen", 2), ("qwen", 8)])
def test_multi_rank_gather_matches_single_rank(tmp_path, model, world):
    path = str(tmp_path / "gathered.pt")
    mp.spawn(_worker, args=(world, _free_port(), path, model), nprocs=world, join=True)
    gathered = torch.load(path)
    single = _local_outputs(0, 1, model)
    bench = _use_model(model)
    assert gathered.shape == single.shape == (bench.HQ, N_SMALL, 128)
    assert torch.equal(gathered, single)
