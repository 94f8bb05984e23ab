"""Sharding and the cross-rank exchange, on CPU with world-size-2 and -3 gloo.

Each rank's chunk partials are the ORACLE's per-path Greeks (the C
restatement of the reference kernel plus the reference's CRN bumps, see
``oracle/__init__.py``) summed per 16384-path chunk -- the same values a
rank's device kernel produces up to fp32 rounding.  What is under test is the
product's host logic: chunk-aligned slicing (Python and the C ABI's
``hmc_slice_chunks`` agree), the exchange in path order, and that the
fixed-order reduction is bit-identical to the single-process one, the
reference's 1-vs-8-workers contract (``tests/test_engine.py:21-32``).
The real kernel under several processes is covered by
``tests/test_gpu_multiprocess.py``."""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2309_10477_b200 import BENCH_PARAMS, HestonParams, OptionSpec, _lib, parallel
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


@pytest.mark.parametrize("n", [1, HMC_CHUNK + 1, 7 * HMC_CHUNK - 3, 2**24, 2**31 + 5])
@pytest.mark.parametrize("world", [1, 2, 3, 5, 8, 16])
def test_c_abi_slice_rule_matches_python(n, world):
    """A C host shards exactly like the Python engine (hmc_slice_chunks)."""
    L = _lib.lib()
    for r in range(world):
        lo, hi = ctypes.c_int64(), ctypes.c_int64()
        assert L.hmc_slice_chunks(n, r, world, ctypes.byref(lo), ctypes.byref(hi)) == 0
        s = parallel.shard(n, r, world)
        assert (lo.value, hi.value) == (s.chunk_lo, s.chunk_hi)
    assert L.hmc_slice_chunks(n, world, world, ctypes.byref(lo), ctypes.byref(hi)) == _lib.HMC_E_INVALID


N_STEPS = 16


def _oracle_chunk_partials(lo, hi, n_runs=2):
    """Per-chunk {sum, sum of squares} of the oracle's seven per-path Greeks
    over paths [lo, hi) (Asian call, 4 fixings, 16 Milstein steps)."""
    import oracle
    p = HestonParams(**BENCH_PARAMS)
    spec = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0,
                      averaging_times=(0.25, 0.5, 0.75, 1.0))
    avg = np.array([4, 8, 12, 16], dtype=np.int64)
    bumps = (0.5, 0.0404, 0.0396, 1e-4)
    out = np.zeros((n_runs, len(range(lo, hi, HMC_CHUNK)), HMC_NW))
    for run in range(n_runs):
        key_run = oracle.derive_key(oracle.root_key(11), run)
        for j, c0 in enumerate(range(lo, hi, HMC_CHUNK)):
            c1 = min(c0 + HMC_CHUNK, hi)
            q = oracle.greeks_paths(p, spec, N_STEPS, True, c0, c1, key_run, None, avg, bumps)
            out[run, j, 0::2] = q.sum(axis=0)
            out[run, j, 1::2] = (q * q).sum(axis=0)
    return torch.tensor(out)


def _seq_reduce(chunks):
    """The device's chunks_to_runs order is fixed by the global chunk count;
    here: sequential over chunks per run (any fixed order proves the point)."""
    c = chunks.numpy()
    return np.array([[sum(c[r, :, w].tolist(), 0.0) for w in range(HMC_NW)] for r in range(c.shape[0])])


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = parallel.shard(n, rank, world)
        local = _oracle_chunk_partials(s.path_lo, s.path_hi)
        full = parallel.gather_chunks(local, n)
        # the surface's int64 histogram exchange (exact integer sums)
        acc = torch.arange(10, dtype=torch.int64) * (rank + 1)
        parallel.allreduce_sum(acc)
        q.put((rank, full.numpy(), acc.numpy()))
    finally:
        torch.distributed.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,n", [(2, 3 * HMC_CHUNK + 77), (2, HMC_CHUNK // 2), (3, 4 * HMC_CHUNK),
                                     (3, 2 * HMC_CHUNK + 5)])
def test_gather_matches_single_process(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {r: (full, acc) for r, full, acc in (q.get(timeout=300) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = _oracle_chunk_partials(0, n).numpy()
    want_acc = np.arange(10) * sum(range(1, world + 1))
    for r in range(world):
        np.testing.assert_array_equal(got[r][0], single)
        np.testing.assert_array_equal(got[r][1], want_acc)
    # and therefore the fixed-order reduction is bit-identical across world sizes
    np.testing.assert_array_equal(_seq_reduce(torch.tensor(got[world - 1][0])),
                                  _seq_reduce(torch.tensor(single)))


def _fallback_worker(rank, world, port, n, q):
    """NCCL-group code path with a libhmc communicator that cannot be
    created: every rank falls back to the group's own collectives."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2309_10477_b200.errors import DeviceError

        def no_comm(group, device):
            raise DeviceError("cannot open libnccl.so.2 (simulated)")
        parallel._uses_nccl = lambda group, tensor: True
        parallel.comm_for = no_comm
        s = parallel.shard(n, rank, world)
        local = torch.arange(s.n_chunks * HMC_NW, dtype=torch.float64).reshape(1, s.n_chunks, HMC_NW)
        local += 1000.0 * s.chunk_lo
        full = parallel.gather_chunks(local, n)
        full2 = parallel.gather_chunks(local, n)        # second call: no retry, same answer
        acc = torch.arange(10, dtype=torch.int64) * (rank + 1)
        parallel.allreduce_sum(acc)
        q.put((rank, full.numpy(), full2.numpy(), acc.numpy(), parallel.comm_fallback_reason()))
    finally:
        torch.distributed.destroy_process_group()


def test_exchange_falls_back_without_libhmc_communicator():
    world, n = 2, 5 * HMC_CHUNK + 9
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fallback_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {r: rest for r, *rest in (q.get(timeout=300) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = []
    for r in range(world):
        s = parallel.shard(n, r, world)
        want.append(np.arange(s.n_chunks * HMC_NW, dtype=np.float64).reshape(1, s.n_chunks, HMC_NW)
                    + 1000.0 * s.chunk_lo)
    want = np.concatenate(want, axis=1)
    for r in range(world):
        full, full2, acc, why = got[r]
        np.testing.assert_array_equal(full, want)
        np.testing.assert_array_equal(full2, want)
        np.testing.assert_array_equal(acc, np.arange(10) * 3)
        assert "simulated" in why
