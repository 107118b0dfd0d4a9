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
