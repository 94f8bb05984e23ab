"""Multi-GPU sharding of the path axis: one process per GPU.

Paths are independent and every per-path value is a pure function of
(seed, run, global path index) -- the reference's determinism contract
(``engine.py:5-9``, ``_core.pyx:385``) -- so the path axis is split into
contiguous, chunk-aligned slices (``HMC_CHUNK`` = 16384 paths), one per rank.
The only exchange is the per-chunk fp64 partials (runs x chunks x 14
doubles, ~100 KB for 2^24 paths): an all-gather over NCCL (NVLink /
NVSwitch), after which every rank reduces the chunks in global path order.
The result is therefore bit-identical for any number of GPUs, extending the
reference's 1-vs-8-workers determinism test (``tests/test_engine.py:21-32``).

The functions here are device-agnostic (they work on any torch tensors and
any initialised process group) so the sharding and gather logic is covered
by world-size-2 ``gloo`` tests on CPU.
"""

from __future__ import annotations

from dataclasses import dataclass

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
    possible (the first ``C % world`` ranks get one more)."""
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


def gather_chunks(local, n_paths: int, group=None):
    """All-gather per-rank chunk partials ``local[run, chunk, HMC_NW]`` into
    the global ``[run, C, HMC_NW]`` tensor in path order (same device/dtype
    as ``local``).  Ranks pad to the largest slice; padding is dropped."""
    import torch
    import torch.distributed as dist
    rank, world = world_info(group)
    if world == 1:
        return local
    n_runs = local.shape[0]
    slices = [shard(n_paths, r, world) for r in range(world)]
    width = max(s.n_chunks for s in slices)
    send = torch.zeros((n_runs, width, HMC_NW), dtype=local.dtype, device=local.device)
    send[:, : local.shape[1]] = local
    recv = torch.empty((world * n_runs, width, HMC_NW), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    recv = recv.view(world, n_runs, width, HMC_NW)
    parts = [recv[r, :, : slices[r].n_chunks] for r in range(world)]
    return torch.cat(parts, dim=1).contiguous()
