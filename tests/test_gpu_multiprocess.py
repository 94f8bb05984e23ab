"""The N>1 path with the REAL kernels: 2 and 3 processes, one gloo group.

Every rank runs the public API (``greeks`` pseudo / Sobol / fp64 replay,
``scheme="exact"``, ``surface``) on its own chunk-aligned slice of the path
axis on ``cuda:0``; the ranks' kernels never wait on one another -- the only
exchange is the chunk partials after the kernels (staged through host
memory, since NCCL refuses two ranks on one GPU).  Every rank's result must
be bit-identical to a single process, the reference's 1-vs-8-workers
contract (``tests/test_engine.py:21-32``) extended across processes.  The
production transport (libhmc's NCCL communicator, one GPU per rank) places
the same bytes in the same order (``hmc_comm_gather_chunks``); its
world-size-1 instance runs in ``test_nccl_comm_world1``.
"""

import ctypes
import os
import socket
import subprocess
import sys
import json

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

CHUNK = 16384


def _jobs():
    from paper_2309_10477_b200 import (BENCH_PARAMS, HestonParams, OptionSpec, SimConfig,
                                       daily_fixings, greeks, surface)
    p = HestonParams(**BENCH_PARAMS)
    euro = OptionSpec("european", "call", 100.0, 1.0, 100.0)
    asian = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0, averaging_times=daily_fixings(1.0, 64))

    def g(spec, **kw):
        base = dict(scheme="milstein", n_paths=5 * CHUNK + 77, n_steps=64, n_runs=2, seed=9)
        base.update(kw)
        res = greeks(p, spec, SimConfig(**base))
        return {q: (s.per_run_values, s.path_std_error) for q, s in res.items()}

    def surf():
        r = surface(p, [90.0, 100.0, 110.0], [0.5, 1.0],
                    SimConfig(scheme="milstein", n_paths=4 * CHUNK + 5, n_steps=64, n_runs=2, seed=3))
        return {f"{st}/{q}": (r.estimate[st][q].tolist(), r.path_std_error[st][q].tolist())
                for st in r.estimate for q in r.estimate[st]}

    return {
        "pseudo_asian": lambda: g(asian),
        "pseudo_euro_3runs": lambda: g(euro, n_runs=3, n_paths=7 * CHUNK),
        "sobol_asian": lambda: g(asian, sampler="sobol", sobol_highdim_ack=True),
        "rqmc_bridge_euro": lambda: g(euro, sampler="sobol", sobol_highdim_ack=True, sobol_scramble=True,
                                      sobol_bridge=8),
        "fp64_asian": lambda: g(asian, precision="fp64", n_paths=2 * CHUNK + 9),
        "exact_euro": lambda: g(euro, scheme="exact", n_steps=1, n_paths=2 * CHUNK + 3),
        "surface": surf,
    }


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    try:
        torch.cuda.set_device(0)
        torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
        out = {name: fn() for name, fn in _jobs().items()}
        q.put((rank, out, None))
        torch.distributed.destroy_process_group()
    except Exception as e:  # noqa: BLE001 - reported to the parent
        import traceback
        q.put((rank, None, traceback.format_exc()))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def single():
    return {name: fn() for name, fn in _jobs().items()}


@pytest.mark.parametrize("world", [2, 3])
def test_multiprocess_bit_identical_to_single_process(single, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        rank, out, err = q.get(timeout=600)
        assert err is None, f"rank {rank}:\n{err}"
        got[rank] = out
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank in range(world):
        for name, want in single.items():
            assert got[rank][name] == want, (world, rank, name)


def test_nccl_comm_world1():
    """libhmc's own NCCL communicator (world 1): init, gather into place for
    1 and 3 runs, int64 all-reduce, destroy."""
    from paper_2309_10477_b200 import _lib
    L = _lib.lib()
    uid = (ctypes.c_uint8 * _lib.HMC_COMM_ID_BYTES)()
    _lib.check(L.hmc_comm_unique_id(uid))
    h = ctypes.c_void_p()
    _lib.check(L.hmc_comm_init(uid, 0, 1, 0, ctypes.byref(h)))
    try:
        s = torch.cuda.current_stream()
        for runs, n in ((1, 3 * CHUNK + 1), (3, 5 * CHUNK)):
            c = -(-n // CHUNK)
            local = torch.randn((runs, c, _lib.HMC_NW), dtype=torch.float64, device="cuda")
            full = torch.full_like(local, float("nan"))
            _lib.check(L.hmc_comm_gather_chunks(h, ctypes.c_void_p(local.data_ptr()), runs, n,
                                                ctypes.c_void_p(full.data_ptr()), ctypes.c_void_p(s.cuda_stream)))
            torch.cuda.synchronize()
            assert torch.equal(full, local)
        acc = torch.arange(100, dtype=torch.int64, device="cuda")
        _lib.check(L.hmc_comm_allreduce_sum(h, ctypes.c_void_p(acc.data_ptr()), 100, _lib.HMC_DTYPE_I64,
                                            ctypes.c_void_p(s.cuda_stream)))
        torch.cuda.synchronize()
        assert torch.equal(acc.cpu(), torch.arange(100, dtype=torch.int64))
    finally:
        _lib.check(L.hmc_comm_destroy(h))


def test_bench_torchrun_two_ranks_gloo():
    """bench.py's N>1 branch under torch.distributed.run, two ranks sharing
    cuda:0 over gloo (HMC_DIST_BACKEND=gloo): one JSON line, n_gpus 2, the
    estimates equal to the single-process engine's."""
    port = _free_port()
    env = dict(os.environ, HMC_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-secondary"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["config"]["parallelism"] == "dp2"
    sys.path.insert(0, ROOT)
    import bench
    from paper_2309_10477_b200 import greeks
    g = greeks(*bench.workload())
    for q, (est, se) in line["estimates"].items():
        assert est == g[q].estimate and se == g[q].path_std_error, q


def _nccl_world1_worker(port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    try:
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        torch.distributed.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
        from paper_2309_10477_b200 import _lib, parallel
        comm = parallel.Comm(None, 0)            # bootstrap: unique id over the NCCL group
        s = torch.cuda.current_stream()
        n = 3 * CHUNK + 5
        local = torch.randn((2, 4, _lib.HMC_NW), dtype=torch.float64, device=dev)
        full = torch.empty_like(local)
        comm.gather_chunks(local, 2, n, full, s)
        acc = torch.arange(7, dtype=torch.int64, device=dev)
        comm.allreduce_sum(acc, s)
        torch.cuda.synchronize()
        ok = torch.equal(full, local) and torch.equal(acc.cpu(), torch.arange(7))
        comm.close()
        torch.distributed.destroy_process_group()
        q.put((ok, None))
    except Exception:  # noqa: BLE001 - reported to the parent
        import traceback
        q.put((False, traceback.format_exc()))


def test_comm_bootstrap_over_nccl_group():
    """parallel.Comm's bootstrap (rank 0's NCCL id over a torch NCCL group)
    and both exchanges, in a world-1 NCCL process group."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_world1_worker, args=(_free_port(), q))
    p.start()
    ok, err = q.get(timeout=300)
    p.join(timeout=60)
    assert ok, err
