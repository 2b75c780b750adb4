"""The device expf (csrc/expf_glibc.cuh) against this host's glibc expf -- the
reference's std::exp(float) (permutation.hpp:171, matrix.hpp:136) -- on ALL
2^32 float inputs, on the box that runs the oracle.

Bit-for-bit for every non-NaN input; NaN inputs must give NaN (the reference
never feeds NaN: tensor_io.hpp rejects non-finite values, and glibc's NaN
payload, x + x on x86, is not an arithmetic result).
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

torch = pytest.importorskip("torch")

CHUNK = 1 << 28


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2510_21270_b200 import ops as _ops

    _ops.lib()
    return _ops


def _host_expf_parallel(x, threads):
    from oracle import host_expf

    parts = np.array_split(x, threads)
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return np.concatenate(list(ex.map(host_expf, parts)))


@pytest.mark.gpu
def test_device_expf_all_2_32_inputs(ops):
    threads = os.cpu_count() or 1
    base = np.arange(CHUNK, dtype=np.uint32)
    mismatches = 0
    examples = []
    for c in range((1 << 32) // CHUNK):
        start = c * CHUNK
        bits = base + np.uint32(start)
        lo = start - (1 << 32) if start >= (1 << 31) else start  # int32 view of the first word
        xd = (torch.arange(CHUNK, dtype=torch.int64, device="cuda") + lo)
        xd = torch.where(xd >= (1 << 31), xd - (1 << 32), xd).to(torch.int32).view(torch.float32)
        dev = ops.debug_expf(xd).view(torch.int32).cpu().numpy().view(np.uint32)
        x = bits.view(np.float32)
        host = _host_expf_parallel(x, threads).view(np.uint32)
        nan_in = np.isnan(x)
        bad = (dev != host) & ~nan_in
        bad |= nan_in & ~np.isnan(dev.view(np.float32))
        nb = int(bad.sum())
        if nb:
            mismatches += nb
            idx = np.flatnonzero(bad)[:3]
            examples += [(hex(int(bits[i])), hex(int(dev[i])), hex(int(host[i]))) for i in idx]
    assert mismatches == 0, f"{mismatches} mismatches (input, device, host): {examples[:6]}"


@pytest.mark.gpu
def test_device_expf_sampled_ranges(ops):
    """Quick variant: random bit patterns plus the exponent ranges the pipeline sees."""
    from oracle import host_expf

    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2**32, size=1 << 24, dtype=np.uint64).astype(np.uint32)
    ranges = [np.linspace(-110.0, 0.0, 1 << 22, dtype=np.float32),
              np.linspace(-1.0, 1.0, 1 << 20, dtype=np.float32),
              np.array([0.0, -0.0, np.inf, -np.inf, 88.72, -103.97, -103.28, -87.3, 1e-30, -1e-30], np.float32)]
    x = np.concatenate([bits.view(np.float32)] + ranges)
    x = x[~np.isnan(x)]
    dev = ops.debug_expf(torch.from_numpy(x).cuda()).cpu().numpy()
    host = host_expf(x)
    bad = np.flatnonzero(dev.view(np.uint32) != host.view(np.uint32))
    assert bad.size == 0, f"{bad.size} mismatches, e.g. x={x[bad[:5]]}"
