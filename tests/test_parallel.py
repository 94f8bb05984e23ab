"""Sharding and the cross-rank exchange, on CPU with world-size-2 gloo.

The kernel is replaced by the oracle (chunk partials computed on the CPU
from per-path Greeks); what is under test is the product's host logic:
chunk-aligned slicing, the all-gather in path order, and that the result is
bit-identical to the single-process reduction."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2309_10477_b200 import parallel
from paper_2309_10477_b200._lib import HMC_CHUNK, HMC_NW


@pytest.mark.parametrize("n", [1, 100, HMC_CHUNK, HMC_CHUNK + 1, 5 * HMC_CHUNK - 3, 2**24])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_covers_axis_once(n, world):
    slices = [parallel.shard(n, r, world) for r in range(world)]
    assert slices[0].path_lo == 0 and slices[-1].path_hi == n
    for a, b in zip(slices, slices[1:]):
        assert a.path_hi == b.path_lo and a.chunk_hi == b.chunk_lo
    for s in slices:
        assert s.path_lo % HMC_CHUNK == 0 or s.n_paths == 0
    assert sum(s.n_chunks for s in slices) == parallel.n_chunks(n)
    sizes = [s.n_chunks for s in slices]
    assert max(sizes) - min(sizes) <= 1


def _chunk_partials(lo, hi, n_runs=2):
    """Stand-in for the device kernel: deterministic pseudo per-path values
    reduced per 16384-path chunk (the same chunking the device uses)."""
    out = []
    for c0 in range(lo, hi, HMC_CHUNK):
        c1 = min(c0 + HMC_CHUNK, hi)
        idx = np.arange(c0, c1, dtype=np.float64)
        row = []
        for run in range(n_runs):
            x = np.sin(idx * 0.001 + run)[:, None] * np.arange(1, HMC_NW // 2 + 1)
            row.append(np.stack([x.sum(0), (x * x).sum(0)], axis=1).reshape(-1))
        out.append(row)
    return torch.tensor(np.array(out).transpose(1, 0, 2).copy()) if out else \
        torch.zeros((n_runs, 0, HMC_NW), dtype=torch.float64)


def _seq_reduce(chunks):
    """The device's chunks_to_runs order: sequential over chunks per run."""
    c = chunks.numpy()
    return np.array([[math.fsum([]) + sum(c[r, :, w].tolist(), 0.0) for w in range(HMC_NW)]
                     for r in range(c.shape[0])])


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = parallel.shard(n, rank, world)
        local = _chunk_partials(s.path_lo, s.path_hi)
        full = parallel.gather_chunks(local, n)
        q.put((rank, full.numpy()))
    finally:
        torch.distributed.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n", [3 * HMC_CHUNK + 77, 4 * HMC_CHUNK, HMC_CHUNK // 2])
def test_gather_world2_matches_single(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = _chunk_partials(0, n).numpy()
    for r in (0, 1):
        np.testing.assert_array_equal(got[r], single)
    # and therefore the fixed-order reduction is bit-identical across G
    np.testing.assert_array_equal(_seq_reduce(torch.tensor(got[1])), _seq_reduce(torch.tensor(single)))

