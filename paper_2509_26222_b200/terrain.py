"""Reference-facing terrain API over the C-ABI.

Mirrors terralio::terrain (/root/reference/proj/core/include/terralio/terrain/
kernel.hpp, center_select.hpp, terrain_model.hpp): same names, argument
meaning and error behaviour (std::invalid_argument -> InvalidArgument,
std::domain_error -> DomainError, NoSupportedCenters, std::runtime_error ->
TerralioError). Every numeric result is computed by the sm_100a kernels in
libterralio_gpu.so; the per-point methods (predict_height, ...) are batches
of one. Batched variants take (m, 2) arrays: numpy (host memory) or torch
CUDA tensors (device memory, results stay on the device).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

from . import _abi
from ._abi import (CenterParamsC, DomainError, InvalidArgument, KernelParamsC,  # noqa: F401
                   NoSupportedCenters, NormalEqC, TerralioError, UpdateReportC, check)

try:  # torch is optional: only needed for device-resident inputs
    import torch
except Exception:  # pragma: no cover
    torch = None


# ---------------------------------------------------------------------------
# kernel.hpp:12-24
@dataclass
class KernelParams:
    sigma: float = 0.04
    sigma_eps: float = 0.1
    lambda_: float = 1e-3
    cutoff_radius: float = 0.0

    def sigma_tilde(self) -> float:
        return math.sqrt(self.sigma * self.sigma + self.sigma_eps * self.sigma_eps)

    def moment_scale(self) -> float:
        st2 = self.sigma * self.sigma + self.sigma_eps * self.sigma_eps
        return self.sigma * self.sigma / st2

    def finalize(self) -> None:
        """KernelParams::finalize (kernel.cpp:15-25)."""
        c = self._c()
        check(_abi.load().tlg_kernel_finalize(C.byref(c)))
        self.cutoff_radius = c.cutoff_radius

    def _c(self) -> KernelParamsC:
        return KernelParamsC(self.sigma, self.sigma_eps, self.lambda_, self.cutoff_radius)

    @staticmethod
    def _from_c(c: KernelParamsC) -> "KernelParams":
        return KernelParams(c.sigma, c.sigma_eps, c.lambda_, c.cutoff_radius)


# types.hpp:14-25
@dataclass
class Rect:
    min: tuple = (0.0, 0.0)
    max: tuple = (0.0, 0.0)

    def contains(self, p) -> bool:
        return self.min[0] <= p[0] <= self.max[0] and self.min[1] <= p[1] <= self.max[1]

    def dilated(self, m: float) -> "Rect":
        return Rect((self.min[0] - m, self.min[1] - m), (self.max[0] + m, self.max[1] + m))


# center_select.hpp:11-28
@dataclass
class TerrainObservation:
    xy: object = None   # (m, 2) numpy or torch CUDA
    z: object = None    # (m,)

    def size(self) -> int:
        return 0 if self.xy is None else len(self.xy)


@dataclass
class CenterSet:
    centers: np.ndarray = field(default_factory=lambda: np.zeros((0, 2)))
    mesh_resolution: float = 0.07
    accept_radius: float = 0.07
    accept_count: int = 3
    roi: Rect = field(default_factory=Rect)

    def _c(self) -> CenterParamsC:
        return CenterParamsC(self.mesh_resolution, self.accept_radius, int(self.accept_count), 0,
                             self.roi.min[0], self.roi.min[1], self.roi.max[0], self.roi.max[1])


class HeightQuery(NamedTuple):
    z: float
    supported: bool


@dataclass
class UpdateReport:
    active_blocks: int = 0
    active_centers: int = 0
    born_centers: int = 0
    rejected: bool = False
    solver: str = ""
    flops: float = 0.0  # FP64 flops of the formulation run (tlg_update_report.flops)


@dataclass
class SparseVec:
    entries: list  # [(id, value)] ascending id


# ---------------------------------------------------------------------------
class Context:
    """A CUDA device + stream for the library (tlg_ctx)."""

    _defaults: dict = {}

    def __init__(self, device: int = 0, stream: int | None = None):
        lib = _abi.load()
        h = C.c_void_p()
        self._follow = stream is None and torch is not None and torch.cuda.is_available()
        if self._follow:
            stream = torch.cuda.current_stream(device).cuda_stream
        # 0 = the legacy default stream (= torch's default stream), never a
        # private one, so inputs torch wrote are ordered before our reads
        check(lib.tlg_ctx_create(int(device), C.c_void_p(stream or 0), C.byref(h)))
        self._handle = h
        self._stream = int(stream or 0)
        self.device = device

    @property
    def handle(self):
        """The tlg_ctx, re-pointed at torch's current stream whenever that
        changed (so calls inside `with torch.cuda.stream(s)` order on s)."""
        if self._follow:
            cur = torch.cuda.current_stream(self.device).cuda_stream
            if cur != self._stream:
                check(_abi.load().tlg_ctx_set_stream(self._handle, C.c_void_p(cur)))
                self._stream = cur
        return self._handle

    def set_stream(self, stream: int) -> None:
        """Pins the context to a raw cudaStream_t (stops following torch)."""
        self._follow = False
        check(_abi.load().tlg_ctx_set_stream(self._handle, C.c_void_p(int(stream))))
        self._stream = int(stream)

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._defaults:
            cls._defaults[device] = Context(device)
        return cls._defaults[device]

    def synchronize(self) -> None:
        check(_abi.load().tlg_ctx_synchronize(self.handle))

    def launch_count(self) -> int:
        return int(_abi.load().tlg_ctx_launch_count(self.handle))

    def __del__(self):
        try:
            if getattr(self, "_handle", None):
                _abi.load().tlg_ctx_destroy(self._handle)
        except Exception:
            pass


# ---------------------------------------------------------------------------
# array plumbing
def _is_dev(a) -> bool:
    return torch is not None and isinstance(a, torch.Tensor) and a.is_cuda


def _col(a, j):
    """Contiguous float64 column j of an (m, 2|3) array, keeping memory space."""
    if _is_dev(a):
        return a[:, j].to(torch.float64).contiguous()
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64)[:, j])


def _vec(a):
    if a is None:
        return None
    if _is_dev(a):
        return a.to(torch.float64).contiguous()
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))


def _ptr(a):
    if a is None:
        return None
    if _is_dev(a):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def _mem(a) -> int:
    return _abi.TLG_DEVICE if _is_dev(a) else _abi.TLG_HOST


def _empty_like(ref, n, dtype):
    if _is_dev(ref):
        tdt = {np.float64: torch.float64, np.uint8: torch.uint8, np.uint32: torch.int32}[dtype]
        return torch.empty(n, dtype=tdt, device=ref.device)
    return np.empty(n, dtype=dtype)


def _xy_of(xy):
    if _is_dev(xy):
        if xy.dim() == 1:
            xy = xy.reshape(1, 2)
        return _col(xy, 0), _col(xy, 1)
    a = np.asarray(xy, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(1, 2)
    return _col(a, 0), _col(a, 1)


def _same_space(*arrs):
    devs = {_is_dev(a) for a in arrs if a is not None}
    if len(devs) > 1:
        raise InvalidArgument("inputs mix host and device memory")


# ---------------------------------------------------------------------------
def kernel_eval(params: KernelParams, x, c, bandwidth: float, ctx: Context | None = None):
    """kernel_eval (kernel.cpp:27-35) on the device, elementwise over (n, 2)
    point and centre arrays (or one pair); DomainError on non-finite input
    or bandwidth <= 0."""
    ctx = ctx or Context.default()
    xs, ys = _xy_of(x)
    cxs, cys = _xy_of(c)
    if len(xs) != len(cxs):
        raise InvalidArgument("x and c differ in length")
    _same_space(xs, cxs)
    out = _empty_like(xs, len(xs), np.float64)
    check(_abi.load().tlg_kernel_eval(ctx.handle, C.byref(params._c()), _ptr(xs), _ptr(ys),
                                      _ptr(cxs), _ptr(cys), len(xs), _mem(xs), float(bandwidth),
                                      _ptr(out), _mem(out)))
    return out


def _nodes_impl(fn_name, obs: TerrainObservation, roi: Rect, res, r_a, count, ctx):
    ctx = ctx or Context.default()
    lib = _abi.load()
    if obs.xy is None:
        xs = ys = np.zeros(0)
    else:
        xs, ys = _xy_of(obs.xy)
    zs = _vec(obs.z) if obs.z is not None else np.zeros(0)
    _same_space(xs, zs)
    cp = CenterSet(mesh_resolution=res, accept_radius=r_a, accept_count=count, roi=roi)._c()
    m, zn = len(xs), len(zs)
    cap = max(16, m)
    n = C.c_size_t(0)
    for _ in range(2):
        ox = np.empty(cap)
        oy = np.empty(cap)
        st = getattr(lib, fn_name)(ctx.handle, _ptr(xs), _ptr(ys), _ptr(zs), m, zn, _mem(xs),
                                   C.byref(cp), _ptr(ox), _ptr(oy), cap, C.byref(n), _abi.TLG_HOST)
        if st == _abi.TLG_BUFFER_TOO_SMALL:
            cap = n.value
            continue
        check(st)
        return np.stack([ox[: n.value], oy[: n.value]], axis=1)
    check(st)


def supported_mesh_nodes(obs: TerrainObservation, roi: Rect, mesh_resolution: float,
                         accept_radius: float, accept_count: int, ctx: Context | None = None):
    """center_select.cpp:18-62 — lattice nodes (i outer, j inner), (k, 2) array."""
    return _nodes_impl("tlg_supported_mesh_nodes", obs, roi, mesh_resolution, accept_radius,
                       accept_count, ctx)


def select_centers(obs: TerrainObservation, roi: Rect, mesh_resolution: float,
                   accept_radius: float, accept_count: int, ctx: Context | None = None) -> CenterSet:
    """center_select.cpp:64-76; raises NoSupportedCenters when empty."""
    nodes = _nodes_impl("tlg_select_centers", obs, roi, mesh_resolution, accept_radius,
                        accept_count, ctx)
    return CenterSet(nodes, mesh_resolution, accept_radius, int(accept_count), roi)


# ---------------------------------------------------------------------------
class _CtxBound:
    """A library handle bound to a Context: reading `handle` first re-points
    the context at torch's current stream (Context.handle)."""

    _h = None

    @property
    def handle(self):
        self.ctx.handle
        return self._h

    @handle.setter
    def handle(self, h):
        self._h = h


class TerrainModel(_CtxBound):
    """terrain_model.hpp:28-97 on the device. Move-only in the reference;
    here a handle that owns the device state."""

    def __init__(self, kernel: KernelParams | None = None, centers: CenterSet | None = None,
                 ctx: Context | None = None, _handle=None):
        self.ctx = ctx or Context.default()
        lib = _abi.load()
        if _handle is not None:
            self.handle = _handle
            return
        kernel = kernel or KernelParams()
        centers = centers or CenterSet()
        c = np.asarray(centers.centers, dtype=np.float64).reshape(-1, 2)
        cx, cy = np.ascontiguousarray(c[:, 0]), np.ascontiguousarray(c[:, 1])
        h = C.c_void_p()
        check(lib.tlg_model_create(self.ctx.handle, C.byref(kernel._c()), C.byref(centers._c()),
                                   _ptr(cx), _ptr(cy), len(cx), _abi.TLG_HOST, C.byref(h)))
        self.handle = h

    def __del__(self):
        try:
            if self._h:
                _abi.load().tlg_model_destroy(self._h)
                self._h = None
        except Exception:
            pass

    # ---- accessors (terrain_model.hpp:33-50) -------------------------------
    def _counts(self):
        nc, nb = C.c_size_t(), C.c_size_t()
        check(_abi.load().tlg_model_counts(self.handle, C.byref(nc), C.byref(nb)))
        return nc.value, nb.value

    def num_centers(self) -> int:
        return self._counts()[0]

    def num_blocks(self) -> int:
        return self._counts()[1]

    def kernel(self) -> KernelParams:
        c = KernelParamsC()
        check(_abi.load().tlg_model_kernel(self.handle, C.byref(c)))
        return KernelParams._from_c(c)

    def centers(self) -> CenterSet:
        lib = _abi.load()
        cp = CenterParamsC()
        check(lib.tlg_model_center_params(self.handle, C.byref(cp)))
        n = self.num_centers()
        cx, cy = np.empty(n), np.empty(n)
        check(lib.tlg_model_get_centers(self.handle, _ptr(cx), _ptr(cy), _abi.TLG_HOST))
        return CenterSet(np.stack([cx, cy], 1), cp.mesh_resolution, cp.accept_radius,
                         cp.accept_count, Rect((cp.roi_min_x, cp.roi_min_y),
                                               (cp.roi_max_x, cp.roi_max_y)))

    def weights(self) -> np.ndarray:
        w = np.empty(self.num_centers())
        check(_abi.load().tlg_model_get_weights(self.handle, _ptr(w), _abi.TLG_HOST))
        return w

    def set_weights(self, w) -> None:
        w = _vec(w)
        check(_abi.load().tlg_model_set_weights(self.handle, _ptr(w), _mem(w)))

    # ---- point-sharded batch ridge -----------------------------
    def batch_system(self) -> tuple[int, int, int]:
        """(n, ld, elems) of the banded batch-ridge system
        (tlg_batch_ridge_system); H holds `elems` doubles."""
        n, ld, el = C.c_size_t(), C.c_size_t(), C.c_size_t()
        check(_abi.load().tlg_batch_ridge_system(self.handle, C.byref(n), C.byref(ld),
                                                 C.byref(el)))
        return n.value, ld.value, el.value

    def batch_pattern(self) -> int:
        """Structural nonzeros of the batch system (tlg_batch_ridge_pattern)."""
        nnz = C.c_size_t()
        check(_abi.load().tlg_batch_ridge_pattern(self.handle, C.byref(nnz)))
        return nnz.value

    def batch_pack(self, H, packed) -> None:
        """packed[:] = the structural nonzeros of device H (tlg_batch_ridge_pack)."""
        if not (_is_dev(H) and _is_dev(packed)):
            raise InvalidArgument("H and packed must be CUDA tensors")
        check(_abi.load().tlg_batch_ridge_pack(self.handle, _ptr(H), _ptr(packed)))

    def batch_unpack(self, packed, H) -> None:
        """H = 0, then the packed entries scattered back (tlg_batch_ridge_unpack)."""
        if not (_is_dev(H) and _is_dev(packed)):
            raise InvalidArgument("H and packed must be CUDA tensors")
        check(_abi.load().tlg_batch_ridge_unpack(self.handle, _ptr(packed), _ptr(H)))

    def batch_assemble(self, xy, z, H, b, add_lambda: bool) -> None:
        """Partial system of this point shard into device tensors H (n * ld)
        and b (n) (tlg_batch_ridge_assemble)."""
        if not (_is_dev(H) and _is_dev(b)):
            raise InvalidArgument("H and b must be CUDA tensors")
        n, ld, el = self.batch_system()
        if H.numel() < el or b.numel() < n:
            raise InvalidArgument("H / b smaller than tlg_batch_ridge_system")
        m = 0 if xy is None else len(xy)
        if m:
            x, y = _xy_of(xy)
            zz = _vec(z)
        else:
            x = y = zz = None
        check(_abi.load().tlg_batch_ridge_assemble(
            self.handle, _ptr(x), _ptr(y), _ptr(zz), m, _mem(x) if m else _abi.TLG_HOST,
            _ptr(H), ld, _ptr(b), 1 if add_lambda else 0))

    def batch_solve(self, H, b) -> None:
        """Factor and solve the (summed) system, writing weights and info_inv
        blocks (tlg_batch_ridge_solve)."""
        n, ld, el = self.batch_system()
        if H.numel() < el or b.numel() < n:
            raise InvalidArgument("H / b smaller than tlg_batch_ridge_system")
        check(_abi.load().tlg_batch_ridge_solve(self.handle, _ptr(H), ld, _ptr(b)))

    def set_exact_cutoff(self, exact: bool = True) -> None:
        """Force the per-pair cutoff test in evaluation (see
        tlg_model_set_exact_cutoff; the default skips it only where provably
        negligible)."""
        check(_abi.load().tlg_model_set_exact_cutoff(self.handle, 1 if exact else 0))

    def sweep(self) -> tuple[int, int]:
        """(sweep kind, exp recurrence used) — tlg_model_sweep."""
        kind, rec = C.c_int(), C.c_int()
        check(_abi.load().tlg_model_sweep(self.handle, C.byref(kind), C.byref(rec)))
        return kind.value, rec.value

    def block_index(self) -> np.ndarray:
        out = np.empty(self.num_centers(), dtype=np.uint32)
        check(_abi.load().tlg_model_get_block_index(self.handle, _ptr(out), _abi.TLG_HOST))
        return out

    def block_of(self, center: int) -> int:
        return int(self.block_index()[center])

    def block_members(self, b: int) -> np.ndarray:
        n = C.c_size_t()
        lib = _abi.load()
        check(lib.tlg_model_block_size(self.handle, int(b), C.byref(n)))
        out = np.empty(n.value, dtype=np.uint32)
        check(lib.tlg_model_get_block_members(self.handle, int(b), _ptr(out)))
        return out

    def block_info_inverse(self, b: int) -> np.ndarray:
        n = C.c_size_t()
        lib = _abi.load()
        check(lib.tlg_model_block_size(self.handle, int(b), C.byref(n)))
        out = np.empty(n.value * n.value)
        check(lib.tlg_model_get_block_info_inverse(self.handle, int(b), _ptr(out), _abi.TLG_HOST))
        return out.reshape(n.value, n.value, order="F")

    def set_block_info_inverse(self, b: int, a) -> None:
        a = np.asfortranarray(np.asarray(a, dtype=np.float64))
        check(_abi.load().tlg_model_set_block_info_inverse(self.handle, int(b), _ptr(a),
                                                            _abi.TLG_HOST))

    # ---- queries -------------------------------------------------------------
    def predict(self, xy, height=True, supported=True, gradient=True):
        """Batched predict_height/predict_gradient: returns (z, supported, gx, gy)
        (entries None when not requested); host in -> numpy out, device in ->
        device tensors out."""
        xs, ys = _xy_of(xy)
        n = len(xs)
        z = _empty_like(xs, n, np.float64) if height else None
        s = _empty_like(xs, n, np.uint8) if supported else None
        gx = _empty_like(xs, n, np.float64) if gradient else None
        gy = _empty_like(xs, n, np.float64) if gradient else None
        check(_abi.load().tlg_eval(self.handle, _ptr(xs), _ptr(ys), n, _mem(xs), _ptr(z), _ptr(s),
                                   _ptr(gx), _ptr(gy), _mem(xs)))
        return z, s, gx, gy

    def export_csv(self, path: str, grid_step: float) -> None:
        """TerrainModel::export_csv (terrain_model.cpp:255-267)."""
        from .consumers import export_csv
        export_csv(self, path, grid_step)

    def predict_height(self, x) -> HeightQuery:
        """terrain_model.cpp:109-125."""
        z, s, _, _ = self.predict(np.asarray(x, dtype=np.float64).reshape(1, 2), gradient=False)
        return HeightQuery(float(z[0]), bool(s[0]))

    def predict_gradient(self, x) -> np.ndarray:
        """terrain_model.cpp:127-143."""
        _, _, gx, gy = self.predict(np.asarray(x, dtype=np.float64).reshape(1, 2), height=False,
                                    supported=False)
        return np.array([gx[0], gy[0]])

    def moment_features(self, xy):
        """Batched moment_feature (terrain_model.cpp:97-107) as CSR
        (row_ptr, ids, vals) with ids ascending per row."""
        xs, ys = _xy_of(xy)
        n = len(xs)
        lib = _abi.load()
        nnz = C.c_size_t(0)
        cap = max(64, n * 80)
        for _ in range(2):
            rp = np.empty(n + 1, dtype=np.uint32)
            ids = np.empty(cap, dtype=np.uint32)
            vals = np.empty(cap)
            st = lib.tlg_moment_features(self.handle, _ptr(xs), _ptr(ys), n, _mem(xs), _ptr(rp),
                                         _ptr(ids), _ptr(vals), cap, C.byref(nnz), _abi.TLG_HOST)
            if st == _abi.TLG_BUFFER_TOO_SMALL:
                cap = nnz.value
                continue
            check(st)
            return rp, ids[: nnz.value], vals[: nnz.value]
        check(st)

    def moment_feature(self, x) -> SparseVec:
        rp, ids, vals = self.moment_features(np.asarray(x, dtype=np.float64).reshape(1, 2))
        return SparseVec([(int(i), float(v)) for i, v in zip(ids, vals)])

    # ---- update (terrain_model.cpp:145-253) ---------------------------------
    def recursive_update(self, obs: TerrainObservation, allow_birth: bool = True) -> UpdateReport:
        if obs.xy is None or len(obs.xy) == 0:
            xs = ys = np.zeros(0)
        else:
            xs, ys = _xy_of(obs.xy)
        zs = _vec(obs.z) if obs.z is not None else np.zeros(0)
        _same_space(xs, zs)
        rep = UpdateReportC()
        check(_abi.load().tlg_recursive_update(self.handle, _ptr(xs), _ptr(ys), _ptr(zs), len(xs),
                                               len(zs), _mem(xs), 1 if allow_birth else 0,
                                               C.byref(rep)))
        return UpdateReport(rep.active_blocks, rep.active_centers, rep.born_centers,
                            bool(rep.rejected), {0: "", 1: "woodbury", 2: "information"}[rep.solver],
                            rep.flops)

    # ---- persistence (snapshot.cpp) ------------------------------------------
    def save(self, path: str) -> None:
        check(_abi.load().tlg_model_save(self.handle, str(path).encode()))

    @staticmethod
    def load(path: str, ctx: Context | None = None) -> "TerrainModel":
        ctx = ctx or Context.default()
        h = C.c_void_p()
        check(_abi.load().tlg_model_load(ctx.handle, str(path).encode(), C.byref(h)))
        return TerrainModel(ctx=ctx, _handle=h)

    def export_csv(self, path: str, grid_step: float) -> None:
        """terrain_model.cpp:255-267: grid "x,y,z_pred", unsupported skipped.
        The grid is evaluated by the batch kernel; only formatting is host-side."""
        roi = self.centers().roi
        xs, x = [], roi.min[0]
        while x <= roi.max[0] + 1e-12:
            xs.append(x)
            x += grid_step
        ys, y = [], roi.min[1]
        while y <= roi.max[1] + 1e-12:
            ys.append(y)
            y += grid_step
        gx, gy = np.meshgrid(np.array(xs), np.array(ys), indexing="ij")
        pts = np.stack([gx.ravel(), gy.ravel()], 1)
        z, s, _, _ = self.predict(pts, gradient=False)
        with open(path, "w") as f:
            f.write("x,y,z_pred\n")
            for (px, py), zz, ok in zip(pts, z, s):
                if ok:
                    f.write(f"{px:.6g},{py:.6g},{zz:.6g}\n")


COMM_ID_BYTES = 128


def comm_unique_id() -> bytes:
    """tlg_comm_unique_id: rank 0 makes it and shares it out of band."""
    buf = C.create_string_buffer(COMM_ID_BYTES)
    check(_abi.load().tlg_comm_unique_id(buf))
    return buf.raw


class Communicator(_CtxBound):
    """tlg_comm (SURVEY §8b tlg_comm_init): the library's own NCCL
    communicator for the sharded variants, one process per GPU."""

    def __init__(self, unique_id: bytes, rank: int, size: int, ctx: Context | None = None):
        self.ctx = ctx or Context.default()
        if len(unique_id) != COMM_ID_BYTES:
            raise InvalidArgument("unique id must be 128 bytes")
        h = C.c_void_p()
        buf = C.create_string_buffer(bytes(unique_id), COMM_ID_BYTES)
        check(_abi.load().tlg_comm_init(self.ctx.handle, buf, int(rank), int(size), C.byref(h)))
        self.handle, self.rank, self.size = h, rank, size

    def allreduce_normal_eq(self, ne):
        """SUM of a kinematics.NormalEq's 29-double block over the ranks."""
        from .kinematics import NormalEq
        c = _abi.NormalEqC()
        c.A[:] = [float(v) for v in np.asarray(ne.A)[np.triu_indices(6)]]
        c.g[:] = [float(v) for v in ne.g]
        c.cost, c.valid = float(ne.cost), float(ne.valid)
        check(_abi.load().tlg_comm_allreduce_normal_eq(self.handle, C.byref(c)))
        return NormalEq._from_c(c)

    def fit_batch_ridge_sharded(self, model: "TerrainModel", xy, z) -> None:
        """tlg_fit_batch_ridge_sharded: this rank's point shard in, the same
        fitted model on every rank out."""
        m = 0 if xy is None else len(xy)
        if m:
            x, y = _xy_of(xy)
            zz = _vec(z)
            mem = _mem(x)
        else:
            x = y = zz = None
            mem = _abi.TLG_HOST
        check(_abi.load().tlg_fit_batch_ridge_sharded(model.handle, self.handle, _ptr(x), _ptr(y),
                                                      _ptr(zz), m, mem))

    def close(self) -> None:
        if self._h is not None:
            _abi.load().tlg_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fit_batch_ridge(kernel: KernelParams, centers: CenterSet, obs: TerrainObservation,
                    ctx: Context | None = None) -> TerrainModel:
    """terrain_model.cpp:269-308."""
    ctx = ctx or Context.default()
    c = np.asarray(centers.centers, dtype=np.float64).reshape(-1, 2)
    cx, cy = np.ascontiguousarray(c[:, 0]), np.ascontiguousarray(c[:, 1])
    if obs.xy is None or len(obs.xy) == 0:
        xs = ys = np.zeros(0)
    else:
        xs, ys = _xy_of(obs.xy)
    zs = _vec(obs.z) if obs.z is not None else np.zeros(0)
    if _is_dev(xs):
        xs, ys, zs = xs.cpu().numpy(), ys.cpu().numpy(), zs.cpu().numpy()
    h = C.c_void_p()
    check(_abi.load().tlg_fit_batch_ridge(ctx.handle, C.byref(kernel._c()), C.byref(centers._c()),
                                          _ptr(cx), _ptr(cy), len(cx), _ptr(xs), _ptr(ys),
                                          _ptr(zs), len(xs), len(zs), _abi.TLG_HOST, C.byref(h)))
    return TerrainModel(ctx=ctx, _handle=h)
