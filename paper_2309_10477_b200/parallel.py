"""Multi-GPU sharding of the path axis: one process per GPU.

Paths are independent and every per-path value is a pure function of
(seed, run, global path index) -- the reference's determinism contract
(``engine.py:5-9``, ``_core.pyx:385``) -- so the path axis is split into
contiguous, chunk-aligned slices (``HMC_CHUNK`` = 16384 paths), one per rank.
The only exchange is the per-chunk fp64 partials (runs x chunks x 14
doubles, ~115 KB for 2^24 paths), after which every rank reduces the chunks
in global path order with the fixed-shape tree.  The result is therefore
bit-identical for any number of GPUs, extending the reference's
1-vs-8-workers determinism test (``tests/test_engine.py:21-32``) and
replacing its fan-out + ordered ``fsum`` (``engine.py:104-116``).

Transport:

* NCCL process groups (one process per GPU, the production layout): the
  exchange runs inside ``libhmc.so`` (``hmc_comm_gather_chunks`` /
  ``hmc_comm_allreduce_sum``, NCCL over NVLink / NVSwitch) on a communicator
  libhmc owns; torch.distributed only bootstraps it (it carries the 128-byte
  NCCL unique id from rank 0 to the others, once per group).
* any other process group (gloo -- the CPU tests, and several ranks sharing
  one GPU, which NCCL refuses): the same partials are staged through host
  memory and exchanged with the group's own collectives.

Both transports place identical bytes in identical order, so the results do
not depend on which one ran.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _lib
from ._lib import HMC_CHUNK, HMC_NW


@dataclass(frozen=True)
class Slice:
    rank: int
    world: int
    path_lo: int
    path_hi: int
    chunk_lo: int
    chunk_hi: int

    @property
    def n_paths(self) -> int:
        return self.path_hi - self.path_lo

    @property
    def n_chunks(self) -> int:
        return self.chunk_hi - self.chunk_lo


def n_chunks(n_paths: int) -> int:
    return (n_paths + HMC_CHUNK - 1) // HMC_CHUNK


def shard(n_paths: int, rank: int, world: int) -> Slice:
    """Rank ``rank``'s contiguous chunk range: chunks are dealt as evenly as
    possible (the first ``C % world`` ranks get one more).  Same rule as the
    C ABI's ``hmc_slice_chunks`` (checked in tests/test_parallel.py)."""
    if not (0 <= rank < world):
        raise ValueError(f"rank {rank} outside world of size {world}")
    C = n_chunks(n_paths)
    base, extra = divmod(C, world)
    c_lo = rank * base + min(rank, extra)
    c_hi = c_lo + base + (1 if rank < extra else 0)
    p_lo = min(c_lo * HMC_CHUNK, n_paths)
    p_hi = min(c_hi * HMC_CHUNK, n_paths)
    return Slice(rank, world, p_lo, p_hi, c_lo, c_hi)


def world_info(group=None) -> tuple[int, int]:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def _uses_nccl(group, tensor) -> bool:
    import torch.distributed as dist
    return tensor.is_cuda and str(dist.get_backend(group)).lower() == "nccl"


# ---------------------------------------------------------------------------
# libhmc communicators (NCCL), one per (process group, device)
# ---------------------------------------------------------------------------
_COMMS: dict = {}


class Comm:
    """A libhmc NCCL communicator spanning the ranks of one process group."""

    def __init__(self, group, device_index: int):
        import torch.distributed as dist
        L = _lib.lib()
        rank, world = world_info(group)
        uid = (ctypes.c_uint8 * _lib.HMC_COMM_ID_BYTES)()
        if rank == 0:
            _lib.check(L.hmc_comm_unique_id(uid))
        box = [bytes(uid)]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(box, src=src, group=group)
        uid = (ctypes.c_uint8 * _lib.HMC_COMM_ID_BYTES).from_buffer_copy(box[0])
        handle = ctypes.c_void_p()
        _lib.check(L.hmc_comm_init(uid, rank, world, device_index, ctypes.byref(handle)))
        self.handle, self.rank, self.world, self.device = handle, rank, world, device_index

    def gather_chunks(self, local, n_runs: int, n_paths: int, full, stream) -> None:
        _lib.check(_lib.lib().hmc_comm_gather_chunks(
            self.handle, ctypes.c_void_p(local.data_ptr() if local.numel() else 0), n_runs, n_paths,
            ctypes.c_void_p(full.data_ptr()), ctypes.c_void_p(stream.cuda_stream)))

    def allreduce_sum(self, buf, stream) -> None:
        import torch
        dtype = {torch.int64: _lib.HMC_DTYPE_I64, torch.float64: _lib.HMC_DTYPE_F64}[buf.dtype]
        _lib.check(_lib.lib().hmc_comm_allreduce_sum(
            self.handle, ctypes.c_void_p(buf.data_ptr()), buf.numel(), dtype,
            ctypes.c_void_p(stream.cuda_stream)))

    def close(self) -> None:
        if self.handle:
            _lib.check(_lib.lib().hmc_comm_destroy(self.handle))
            self.handle = None


def comm_for(group, device) -> Comm:
    """The libhmc communicator of ``group`` on ``device`` (created on first
    use -- a collective call on every rank of the group)."""
    key = (id(group) if group is not None else None, device.index)
    c = _COMMS.get(key)
    if c is None or c.handle is None:
        c = Comm(group, device.index)
        _COMMS[key] = c
    return c


def close_comms() -> None:
    """Destroy every libhmc communicator (before destroy_process_group)."""
    for c in _COMMS.values():
        c.close()
    _COMMS.clear()


# ---------------------------------------------------------------------------
# the exchanges the engine uses
# ---------------------------------------------------------------------------
# (process group, device) pairs whose libhmc communicator could not be
# created: their exchanges go through the group's own collectives (the same
# bytes in the same order), reported once on stderr
_COMM_FAILED: dict = {}


def comm_fallback_reason(group=None, device_index=None):
    """Why the libhmc communicator of (group, device) is not in use, or None."""
    if device_index is None:
        return next(iter(_COMM_FAILED.values()), None)
    return _COMM_FAILED.get((id(group) if group is not None else None, device_index))


def _libhmc_comm(group, device):
    """The group's libhmc communicator, or None if it cannot be created (then
    every rank of the group falls back to the group's collectives: a failure
    to open or initialise NCCL is the same on every rank)."""
    import sys
    from .errors import HestonError
    key = (id(group) if group is not None else None, device.index)
    if key in _COMM_FAILED:
        return None
    try:
        return comm_for(group, device)
    except HestonError as e:
        _COMM_FAILED[key] = str(e)
        print(f"paper_2309_10477_b200.parallel: libhmc NCCL communicator unavailable ({e}); "
              "exchanging chunk partials through the process group instead", file=sys.stderr)
        return None


def gather_chunks(local, n_paths: int, group=None):
    """All-gather per-rank chunk partials ``local[run, chunk, HMC_NW]`` into
    the global ``[run, C, HMC_NW]`` tensor in path order (same device/dtype
    as ``local``), identical on every rank."""
    import torch
    rank, world = world_info(group)
    if world == 1:
        return local
    n_runs = local.shape[0]
    C = n_chunks(n_paths)
    if _uses_nccl(group, local):
        comm = _libhmc_comm(group, local.device)
        if comm is not None:
            full = torch.empty((n_runs, C, HMC_NW), dtype=local.dtype, device=local.device)
            stream = torch.cuda.current_stream(local.device)
            comm.gather_chunks(local.contiguous(), n_runs, n_paths, full, stream)
            return full
        return _gather_chunks_group(local, n_paths, group, on_device=True)
    return _gather_chunks_group(local, n_paths, group, on_device=False)


def _gather_chunks_group(local, n_paths: int, group=None, on_device: bool = False):
    """The process group's own all-gather of padded slices (gloo: staged
    through host memory; NCCL without a libhmc communicator: on the device),
    padding dropped, concatenated in rank (= path) order."""
    import torch
    import torch.distributed as dist
    rank, world = world_info(group)
    n_runs = local.shape[0]
    slices = [shard(n_paths, r, world) for r in range(world)]
    width = max(s.n_chunks for s in slices)
    dev = local.device if on_device else torch.device("cpu")
    send = torch.zeros((n_runs, width, HMC_NW), dtype=local.dtype, device=dev)
    send[:, : local.shape[1]] = local.to(dev)
    recv = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(recv, send, group=group)
    parts = [recv[r][:, : slices[r].n_chunks] for r in range(world)]
    return torch.cat(parts, dim=1).contiguous().to(local.device)


def _gather_chunks_host(local, n_paths: int, group=None):
    """The gloo transport (host-staged)."""
    return _gather_chunks_group(local, n_paths, group, on_device=False)


def allreduce_sum(buf, group=None) -> None:
    """In-place sum over the group's ranks (the surface's int64 histograms:
    integer addition, so exact in any order)."""
    import torch
    import torch.distributed as dist
    _, world = world_info(group)
    if world == 1:
        return
    if _uses_nccl(group, buf):
        comm = _libhmc_comm(group, buf.device)
        if comm is not None:
            comm.allreduce_sum(buf, torch.cuda.current_stream(buf.device))
        else:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        return
    host = buf.cpu()
    dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
    buf.copy_(host)
