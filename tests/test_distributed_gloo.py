"""world_size-2 gloo test of the sharded manifold-row reduction: every rank
evaluates its contiguous shard (CPU oracle stands in for the device kernel)
and allreduce_normal_eq must reproduce the single-process normal equations."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _field():
    sys.path[:0] = [str(ROOT), str(ROOT / "tests"), str(ROOT / "oracle")]
    import oracle as orc
    from helpers import make_field, uniform_xy
    k, cs, obs = make_field(31, 900)
    m = orc.fit_batch_ridge(k, cs, obs.xy, obs.z)
    R = orc.so3_exp([0.02, -0.015, 0.04])
    t = np.array([0.1, -0.05, 0.08])
    pts = np.concatenate([uniform_xy(orc.Rng(9), 3001, -0.1, 1.1), np.full((3001, 1), 0.05)], 1)
    return m, R, t, (pts - t) @ R


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_26222_b200 import distributed as D
    m, R, t, h = _field()
    b, e = D.shard_range(len(h), rank, world)
    _, ne29 = m.manifold_rows(R, t, h[b:e], 0.0, 1.0, 0.05)
    tot = D.allreduce_normal_eq(D.unpack(ne29))
    out[rank] = D.pack(tot).tolist()
    dist.destroy_process_group()


def test_shard_range_covers():
    from paper_2509_26222_b200.distributed import shard_range
    for n in (0, 1, 7, 3001):
        for w in (1, 2, 3, 8):
            r = [shard_range(n, k, w) for k in range(w)]
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(r[i][1] == r[i + 1][0] for i in range(w - 1))


def test_gloo_allreduce_matches_single_process():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    m, R, t, h = _field()
    _, ne = m.manifold_rows(R, t, h, 0.0, 1.0, 0.05)
    for rank in range(2):
        got = np.array(out[rank])
        np.testing.assert_allclose(got[:28], ne[:28], rtol=1e-12, atol=1e-12 * np.abs(ne).max())
        assert got[28] == ne[28]


class _DenseRidge:
    """CPU stand-in for TerrainModel's batch_system / batch_assemble /
    batch_solve (dense numpy, Gaussian features of fixed centres): checks the
    sharded driver's plumbing — lambda added once, partial systems summed,
    every rank solving the same system."""

    def __init__(self, lam=1e-3):
        g = np.linspace(0.0, 1.0, 6)
        self.c = np.array([(a, b) for a in g for b in g])
        self.lam = lam
        self.w = None

    def batch_system(self):
        return len(self.c), len(self.c), len(self.c) ** 2

    def _feat(self, xy):
        d2 = ((xy[:, None, :] - self.c[None, :, :]) ** 2).sum(-1)
        return np.exp(-d2 / (2 * 0.2 ** 2))

    def batch_assemble(self, xy, z, H, b, add_lambda):
        import torch
        n = len(self.c)
        M = self._feat(np.asarray(xy)) if xy is not None and len(xy) else np.zeros((0, n))
        Hn = M.T @ M + (self.lam * np.eye(n) if add_lambda else 0.0)
        bn = M.T @ (np.asarray(z) if len(M) else np.zeros(0))
        H.copy_(torch.from_numpy(np.ascontiguousarray(Hn.T).reshape(-1)))
        b.copy_(torch.from_numpy(bn))

    def batch_solve(self, H, b):
        n = len(self.c)
        self.w = np.linalg.solve(H.numpy().reshape(n, n).T, b.numpy())


class _PackedRidge(_DenseRidge):
    """+ the packed reduction hooks: entries of centre pairs farther apart
    than 0.5 are structurally zero (a band of the dense system), packed in a
    fixed order."""

    def _pos(self):
        d = np.linalg.norm(self.c[:, None, :] - self.c[None, :, :], axis=-1)
        return np.flatnonzero((d <= 0.5).reshape(-1))

    def batch_pattern(self):
        return len(self._pos())

    def batch_pack(self, H, P):
        import torch
        P.copy_(H[torch.from_numpy(self._pos())])

    def batch_unpack(self, P, H):
        import torch
        H.zero_()
        H[torch.from_numpy(self._pos())] = P


def _ridge_data():
    rng = np.random.default_rng(3)
    xy = rng.uniform(0.0, 1.0, (501, 2))
    return xy, np.sin(3 * xy[:, 0]) * xy[:, 1]


def _ridge_worker(rank, world, port, out, packed=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
    from paper_2509_26222_b200 import distributed as D
    from test_distributed_gloo import _DenseRidge, _PackedRidge, _ridge_data
    xy, z = _ridge_data()
    b, e = D.shard_range(len(z), rank, world)
    m = _PackedRidge() if packed else _DenseRidge()
    _, _, moved = D.fit_batch_ridge_sharded(m, xy[b:e], z[b:e], device="cpu")
    out[rank] = m.w.tolist()
    out[f"moved{rank}"] = moved
    dist.destroy_process_group()


def test_gloo_sharded_batch_ridge_matches_single_process():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_ridge_worker, args=(2, port, out), nprocs=2, join=True)
    xy, z = _ridge_data()
    ref = _DenseRidge()
    from paper_2509_26222_b200 import distributed as D
    D.fit_batch_ridge_sharded(ref, xy, z, device="cpu")
    for rank in range(2):
        np.testing.assert_allclose(np.array(out[rank]), ref.w, rtol=1e-9, atol=1e-12)
    assert out[0] == out[1]


def test_gloo_sharded_batch_ridge_packed_reduction():
    """The packed (structural-nonzero) reduction gives the same system as the
    dense one when the dropped entries are zero in every partial system."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_ridge_worker, args=(2, port, out, True), nprocs=2, join=True)
    xy, z = _ridge_data()
    ref = _PackedRidge()
    n = len(ref.c)
    # the single-process reference on the same pattern-restricted system
    import torch
    H = torch.empty(n * n, dtype=torch.float64)
    b = torch.empty(n, dtype=torch.float64)
    ref.batch_assemble(xy, z, H, b, True)
    P = torch.empty(ref.batch_pattern(), dtype=torch.float64)
    ref.batch_pack(H, P)
    ref.batch_unpack(P, H)
    ref.batch_solve(H, b)
    for rank in range(2):
        np.testing.assert_allclose(np.array(out[rank]), ref.w, rtol=1e-9, atol=1e-12)
        assert out[f"moved{rank}"] == ref.batch_pattern() + n < n * n + n
    assert out[0] == out[1]
