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


def _local_outputs(rank, world):
    import bench
    import oracle

    kv0, kv_local, q0, hq_local = bench.shard_of(rank, world)
    q, k, v = bench.make_inputs(torch, N_SMALL, hq_local, kv_local, kv0, "cpu")
    orc = oracle.Oracle("oracle")
    cfg = oracle.make_config(block_size=64, segment_size=128, tau=0.9, strategy="key_permute")
    g = bench.HQ // bench.HKV
    outs = []
    for h in range(hq_local):
        r = orc.pbs_attention(q[h].float().numpy(), k[h // g].float().numpy(), v[h // g].float().numpy(), cfg)
        outs.append(torch.from_numpy(r.output))
    return torch.stack(outs)


def _worker(rank, world, port, path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = _local_outputs(rank, world)
    full = [torch.empty_like(out) for _ in range(world)]
    dist.all_gather(full, out)
    if rank == 0:
        torch.save(torch.cat(full), path)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_arithmetic():
    import bench

    for world in (1, 2, 4, 8):
        owned = []
        for r in range(world):
            kv0, kvl, q0, ql = bench.shard_of(r, world)
            assert ql == kvl * (bench.HQ // bench.HKV) and q0 == kv0 * (bench.HQ // bench.HKV)
            owned += list(range(q0, q0 + ql))
        assert owned == list(range(bench.HQ))
    with pytest.raises(ValueError):
        bench.shard_of(0, 3)


def test_two_rank_gather_matches_single_rank(tmp_path):
    path = str(tmp_path / "gathered.pt")
    mp.spawn(_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    gathered = torch.load(path)
    single = _local_outputs(0, 1)
    assert gathered.shape == single.shape == (32, N_SMALL, 128)
    assert torch.equal(gathered, single)
