"""Multi-GPU execution by right-hand side.

Sources are independent, so the path shards by RHS. Every rank (one process per
GPU) holds a full replica of the factors and solves its own slice of the sources.
There is no exchange during a solve. Rank 0 gathers the wavefields at the end;
the gather runs over NCCL/NVLink on GPUs, or gloo in tests.
"""

from __future__ import annotations

import numpy as np

__all__ = ["source_slice", "solve_sharded", "gather_to_root"]


def source_slice(n_sources, world, rank):
    """Contiguous near-equal slice of source indices owned by ``rank`` (remainder first)."""
    base, rem = divmod(n_sources, world)
    lo = rank * base + min(rank, rem)
    return range(lo, lo + base + (1 if rank < rem else 0))


def gather_to_root(local, n_sources, group=None):
    """Gather per-rank ``(indices, arrays)`` to rank 0 as one ``[n_sources, ...]`` array."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    objs = [None] * world if rank == 0 else None
    dist.gather_object(local, objs, dst=0, group=group)
    if rank != 0:
        return None
    first = next(a for idx, a in objs if len(idx))
    out = np.empty((n_sources,) + first.shape[1:], dtype=first.dtype)
    for idx, arr in objs:
        for k, i in enumerate(idx):
            out[i] = arr[k]
    return out


def solve_sharded(solve_many, F, group=None):
    """Solve ``F[n, wz, wx]`` across the ranks of ``group``.

    ``solve_many(F_local) -> U_local``: the per-rank solver, e.g.
    ``lambda F: np.stack([r.u for r in solver.solve_many(F)])``.  Returns the
    gathered wavefields on rank 0 and ``None`` elsewhere.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    idx = list(source_slice(F.shape[0], world, rank))
    U = solve_many(F[idx]) if idx else np.zeros((0,) + F.shape[1:], dtype=np.complex128)
    return gather_to_root((idx, U), F.shape[0], group)
