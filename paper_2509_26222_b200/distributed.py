"""Multi-GPU plumbing for the point-sharded paths.

One process per GPU (torch.distributed, NCCL over NVLink on the B200 box;
gloo works for the CPU tests). Points are sharded contiguously.

* Manifold rows: every rank evaluates its shard with tlg_manifold_rows /
  tlg_scan_manifold_rows; the only data-path exchange is the 29-double
  normal-equation block (J^T J upper 21, J^T r 6, cost, valid) summed across
  ranks — the one real reduction of the LM cost evaluation.
* Batch ridge (kernel-matrix assembly): every rank assembles the banded
  partial system (lambda I on rank 0) + sum m m^T, sum m z over its shard
  (tlg_batch_ridge_assemble); the structural nonzeros of the band
  (tlg_batch_ridge_pack: centre pairs within two cutoffs, ~4% of the band
  storage at C5) and the rhs are summed across ranks, unpacked, and every
  rank factors and solves the same system ("replicas" for the solve,
  SURVEY §8e).
"""
from __future__ import annotations

import numpy as np

from .kinematics import NormalEq

_IU = np.triu_indices(6)


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [b, e) of n points for `rank` (sizes differ by <= 1)."""
    base, extra = divmod(n, world)
    b = rank * base + min(rank, extra)
    return b, b + base + (1 if rank < extra else 0)


def pack(ne: NormalEq) -> np.ndarray:
    return np.concatenate([ne.A[_IU], ne.g, [ne.cost, float(ne.valid)]])


def unpack(v) -> NormalEq:
    v = np.asarray(v, dtype=np.float64)
    A = np.zeros((6, 6))
    A[_IU] = v[:21]
    A = A + A.T - np.diag(np.diag(A))
    return NormalEq(A, v[21:27].copy(), float(v[27]), int(round(v[28])))


def allreduce_normal_eq(ne: NormalEq, group=None, device=None, buf=None) -> NormalEq:
    """Sums the normal equations over all ranks (torch.distributed SUM).

    `buf` may be a preallocated 29-element float64 tensor on `device` (the
    bench keeps one on the GPU so NCCL reduces device memory)."""
    import torch
    import torch.distributed as dist

    v = torch.from_numpy(pack(ne))
    if buf is None:
        buf = v.to(device) if device is not None else v
    else:
        buf.copy_(v)
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return unpack(buf.cpu().numpy())


def fit_batch_ridge_sharded(model, xy_shard, z_shard, group=None, device=None, packed=True):
    """Point-sharded fit_batch_ridge into `model` (created from the same
    centres on every rank). `model` needs batch_system / batch_assemble /
    batch_solve (terrain.TerrainModel on the GPU). Returns (n, ld, moved):
    the reduced system's size (band storage, TerrainModel.batch_system) and
    the doubles each rank contributed to the reduction.

    The partial systems are reduced in PACKED form when the model offers
    batch_pattern / batch_pack / batch_unpack: only the structural nonzeros
    (centre pairs within two cutoffs, the same deterministic order on every
    rank) cross NVLink — C5: ~1.3e7 doubles instead of the 3.4e8 of the band
    storage — then every rank unpacks and solves the same system."""
    import torch
    import torch.distributed as dist

    on = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank(group) if on else 0
    n, ld, elems = model.batch_system()
    dev = device or ("cuda" if torch.cuda.is_available() else "cpu")
    H = torch.empty(elems, dtype=torch.float64, device=dev)
    b = torch.empty(n, dtype=torch.float64, device=dev)
    model.batch_assemble(xy_shard, z_shard, H, b, add_lambda=(rank == 0))
    moved = elems + n
    if on:
        use_packed = packed and hasattr(model, "batch_pattern")
        nnz = model.batch_pattern() if use_packed else elems
        if use_packed and nnz < elems:
            P = torch.empty(nnz, dtype=torch.float64, device=dev)
            model.batch_pack(H, P)
            dist.all_reduce(P, op=dist.ReduceOp.SUM, group=group)
            model.batch_unpack(P, H)
            moved = nnz + n
        else:
            dist.all_reduce(H, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(b, op=dist.ReduceOp.SUM, group=group)
    model.batch_solve(H, b)
    return n, ld, moved
