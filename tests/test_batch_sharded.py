"""Batch ridge in band storage and its point-sharded form:
tlg_fit_batch_ridge on a field large enough that the banded system is
stored in band form (ld < n) against the oracle's dense LDLT
(terrain_model.cpp:269-308), and the assemble / sum / solve split — two
shards emulated on one GPU, and the world-1 driver — against the single-call
fit."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle as orc
from helpers import rel_norm, uniform_xy
from paper_2509_26222_b200 import distributed as D
from paper_2509_26222_b200 import terrain as T

pytestmark = pytest.mark.gpu


def _field(side=2.2, n_points=6000, seed=41):
    k = T.KernelParams(sigma=0.04, sigma_eps=0.1)
    k.finalize()
    xy = uniform_xy(orc.Rng(seed), n_points, 0.0, side)
    z = 0.1 * np.sin(4.0 * xy[:, 0]) + 0.05 * xy[:, 1] ** 2
    roi = T.Rect((0.0, 0.0), (side, side))
    nodes = orc.supported_mesh_nodes(xy, z, roi, 0.07, 0.12, 3)
    return k, T.CenterSet(nodes, 0.07, 0.12, 3, roi), T.TerrainObservation(xy, z)


def test_batch_fit_band_storage_parity(gpu_ctx):
    k, cs, obs = _field()
    g = T.fit_batch_ridge(k, cs, obs)
    n, ld, el = g.batch_system()
    assert n == len(cs.centers) and ld < n and el == n * (ld + 1)  # band storage in use
    o = orc.fit_batch_ridge(k, cs, obs.xy, obs.z)
    assert rel_norm(g.weights(), o.weights()) < 1e-8
    for b in range(o.num_blocks()):
        assert rel_norm(g.block_info_inverse(b), o.block_info_inverse(b)) < 1e-8


def test_batch_fit_two_shards_equal_single_call(gpu_ctx):
    k, cs, obs = _field(seed=42)
    full = T.fit_batch_ridge(k, cs, obs)
    g = T.TerrainModel(k, cs)
    n, ld, el = g.batch_system()
    cut = len(obs.z) // 3
    parts = []
    for r, (b0, b1) in enumerate(((0, cut), (cut, len(obs.z)))):
        H = torch.empty(el, dtype=torch.float64, device="cuda")
        b = torch.empty(n, dtype=torch.float64, device="cuda")
        g.batch_assemble(obs.xy[b0:b1], obs.z[b0:b1], H, b, add_lambda=(r == 0))
        parts.append((H, b))
    H = parts[0][0] + parts[1][0]
    b = parts[0][1] + parts[1][1]
    g.batch_solve(H, b)
    assert rel_norm(g.weights(), full.weights()) < 1e-10
    for q in range(full.num_blocks()):
        assert rel_norm(g.block_info_inverse(q), full.block_info_inverse(q)) < 1e-10


def test_batch_fit_sharded_world1_bit_identical(gpu_ctx):
    k, cs, obs = _field(side=1.2, n_points=2500, seed=43)
    full = T.fit_batch_ridge(k, cs, obs)
    g = T.TerrainModel(k, cs)
    D.fit_batch_ridge_sharded(g, obs.xy, obs.z)
    assert np.array_equal(g.weights(), full.weights())


def test_batch_assemble_empty_shard(gpu_ctx):
    k, cs, obs = _field(side=1.2, n_points=2500, seed=44)
    g = T.TerrainModel(k, cs)
    n, ld, el = g.batch_system()
    H = torch.full((el,), 7.0, dtype=torch.float64, device="cuda")
    b = torch.full((n,), 7.0, dtype=torch.float64, device="cuda")
    g.batch_assemble(None, None, H, b, add_lambda=False)
    assert float(H.abs().max()) == 0.0 and float(b.abs().max()) == 0.0


def test_batch_pack_unpack_roundtrip_exact(gpu_ctx):
    """Every nonzero of an assembled partial system lies in the packed
    pattern (pair distance <= two cutoffs): unpack(pack(H)) == H bit for bit,
    and the pattern is a small fraction of the band storage."""
    k, cs, obs = _field(seed=45)
    g = T.TerrainModel(k, cs)
    n, ld, el = g.batch_system()
    H = torch.empty(el, dtype=torch.float64, device="cuda")
    b = torch.empty(n, dtype=torch.float64, device="cuda")
    g.batch_assemble(obs.xy, obs.z, H, b, add_lambda=True)
    nnz = g.batch_pattern()
    assert n <= nnz < el
    P = torch.empty(nnz, dtype=torch.float64, device="cuda")
    g.batch_pack(H, P)
    H2 = torch.full((el,), 3.0, dtype=torch.float64, device="cuda")
    g.batch_unpack(P, H2)
    assert torch.equal(H, H2)


def test_batch_fit_two_shards_packed_equal_dense_sum(gpu_ctx):
    """The packed reduction (pack, sum the packed vectors, unpack) yields the
    same summed system as adding the band storage, so the fit is bit-identical
    to the dense-sum path and within 1e-10 of the single call."""
    k, cs, obs = _field(seed=46)
    full = T.fit_batch_ridge(k, cs, obs)
    g = T.TerrainModel(k, cs)
    n, ld, el = g.batch_system()
    nnz = g.batch_pattern()
    cut = len(obs.z) // 3
    Hs, bs, Ps = [], [], []
    for r, (b0, b1) in enumerate(((0, cut), (cut, len(obs.z)))):
        H = torch.empty(el, dtype=torch.float64, device="cuda")
        b = torch.empty(n, dtype=torch.float64, device="cuda")
        g.batch_assemble(obs.xy[b0:b1], obs.z[b0:b1], H, b, add_lambda=(r == 0))
        P = torch.empty(nnz, dtype=torch.float64, device="cuda")
        g.batch_pack(H, P)
        Hs.append(H), bs.append(b), Ps.append(P)
    Hsum = torch.empty(el, dtype=torch.float64, device="cuda")
    g.batch_unpack(Ps[0] + Ps[1], Hsum)
    assert torch.equal(Hsum, Hs[0] + Hs[1])
    g.batch_solve(Hsum, bs[0] + bs[1])
    assert rel_norm(g.weights(), full.weights()) < 1e-10


def _assemble(g, obs, csr):
    from paper_2509_26222_b200 import _abi
    _abi.check(_abi.load_diag().tlg_diag_set_batch_gram(g.handle, 1 if csr else 0))
    n, ld, el = g.batch_system()
    H = torch.empty(el, dtype=torch.float64, device="cuda")
    b = torch.empty(n, dtype=torch.float64, device="cuda")
    g.batch_assemble(obs.xy, obs.z, H, b, add_lambda=True)
    return H, b


@pytest.mark.parametrize("sigma,sigma_eps,side,holes", [(0.04, 0.1, 2.2, 0.0), (None, None, 1.6, 0.0),
                                                       (None, None, 1.6, 0.15), (0.03, 0.05, 1.3, 0.1)])
def test_batch_lattice_assembly_matches_csr_gram(gpu_ctx, sigma, sigma_eps, side, holes):
    """The lattice element assembly (assemble.cu: per-cell DMMA Gram of the
    dense feature block) gives the row-wise CSR Gram's system to rounding —
    the same pair membership, summed in another order — on the paper's
    geometry, other windows and lattices with holes (absent nodes)."""
    k = T.KernelParams() if sigma is None else T.KernelParams(sigma=sigma, sigma_eps=sigma_eps)
    k.finalize()
    rng = np.random.default_rng(47)
    xy = rng.uniform(0.0, side, (40_000, 2))
    z = 0.1 * np.sin(4.0 * xy[:, 0]) + 0.05 * xy[:, 1] ** 2
    roi = T.Rect((0.0, 0.0), (side, side))
    nodes = orc.supported_mesh_nodes(xy, z, roi, 0.07, 0.12, 3)
    if holes:
        nodes = nodes[rng.uniform(size=len(nodes)) >= holes]
    cs = T.CenterSet(nodes, 0.07, 0.12, 3, roi)
    # observations beyond the ROI too (windows leaving the lattice)
    oxy = np.concatenate([xy, rng.uniform(-0.5, side + 0.5, (3000, 2))])
    obs = T.TerrainObservation(oxy, np.concatenate([z, rng.normal(0, 0.1, 3000)]))
    g = T.TerrainModel(k, cs)
    assert g.sweep()[0] != 0  # a lattice
    H1, b1 = _assemble(g, obs, csr=False)
    from paper_2509_26222_b200 import _abi
    used = C.c_int()
    _abi.check(_abi.load_diag().tlg_diag_last_gram_lattice(g.handle, C.byref(used)))
    assert used.value == 1  # the lattice path ran
    H0, b0 = _assemble(g, obs, csr=True)
    assert float((H1 - H0).abs().max()) <= 1e-12 * float(H0.abs().max())
    assert float((b1 - b0).abs().max()) <= 1e-12 * float(b0.abs().max())
    assert torch.equal(H1 == 0, H0 == 0)  # the same structural pattern
    # bit-reproducible run to run
    H2, b2 = _assemble(g, obs, csr=False)
    assert torch.equal(H1, H2) and torch.equal(b1, b2)


def test_comm_world1_sharded_fit_and_normal_eq(gpu_ctx):
    """tlg_comm: a one-rank NCCL communicator from the library's
    own entry points; the sharded fit equals tlg_fit_batch_ridge bit for bit
    and the normal-equation reduction is the identity."""
    from paper_2509_26222_b200 import kinematics as kin
    k, cs, obs = _field(side=1.2, n_points=2500, seed=48)
    full = T.fit_batch_ridge(k, cs, obs)
    comm = T.Communicator(T.comm_unique_id(), 0, 1)
    g = T.TerrainModel(k, cs)
    comm.fit_batch_ridge_sharded(g, obs.xy, obs.z)
    assert np.array_equal(g.weights(), full.weights())
    for b in range(full.num_blocks()):
        assert np.array_equal(g.block_info_inverse(b), full.block_info_inverse(b))
    rng = np.random.default_rng(2)
    A = rng.normal(size=(6, 6))
    ne = kin.NormalEq(A @ A.T, rng.normal(size=6), 3.5, 17)
    out = comm.allreduce_normal_eq(ne)
    assert np.array_equal(out.A, ne.A) and np.array_equal(out.g, ne.g) and out.valid == 17
    comm.close()


def test_information_form_beyond_25600_centres(gpu_ctx):
    """The information-form update on more than 25,600 active centres (the
    banded Gram's window, not n, bounds it): one update from the prior equals
    fit_batch_ridge on the same observations (test_terrain_model.cpp's
    recursive == batch property) to 1e-8."""
    k = T.KernelParams()
    k.finalize()
    side = 169 * 0.07
    nodes = np.arange(170) * 0.07
    gx, gy = np.meshgrid(nodes, nodes, indexing="ij")
    roi = T.Rect((0.0, 0.0), (side, side))
    cs = T.CenterSet(np.stack([gx.ravel(), gy.ravel()], 1), 0.07, 0.12, 3, roi)
    rng = np.random.default_rng(52)
    xy = rng.uniform(0.0, side, (60_000, 2))
    z = 0.05 * np.sin(2.0 * xy[:, 0]) * np.cos(1.5 * xy[:, 1])
    obs = T.TerrainObservation(xy, z)
    g = T.TerrainModel(k, cs)
    rep = g.recursive_update(obs, False)
    assert rep.solver == "information" and rep.active_centers > 25_600, rep
    full = T.fit_batch_ridge(k, cs, obs)
    assert rel_norm(g.weights(), full.weights()) < 1e-8
    # the updated blocks are diagonal blocks of H^-1 (the batch fit stores
    # (H_bb)^-1 instead, so they are not compared): symmetric positive
    # definite and below the prior lambda^-1 I
    for b in range(0, g.num_blocks(), max(1, g.num_blocks() // 7)):
        P = g.block_info_inverse(b)
        assert np.array_equal(P, P.T)
        ev = np.linalg.eigvalsh(P)
        assert ev.min() > 0.0 and ev.max() <= 1.0 / k.lambda_ * (1 + 1e-9)
