"""TEST INFRASTRUCTURE — ctypes wrapper of the CPU oracle (liboracle.so).

The oracle is a plain-C++ restatement of the reference hot path (see
terralio_oracle.hpp). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module; it is the
checker, never the product path.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ODIR = Path(__file__).resolve().parent
LIB = ODIR / "_build" / "liboracle.so"
# The reference itself, compiled from /root/reference by `make -C oracle ref`
# (oracle/ref_capi.cpp exposes it through the same orc_* entry points).
REF_LIB = ODIR / "_ref" / "libterralio_ref.so"
REFERENCE_SRC = Path("/root/reference/proj/core/src")
BACKEND = "port"
_REF_MODULE = None


def reference():
    """This module's API bound to the compiled reference (oracle/_ref), or None
    when it is not built here and cannot be (no /root/reference). Functions
    the reference keeps file-local raise OracleError(UNSUPPORTED)."""
    global _REF_MODULE
    if _REF_MODULE is None:
        if not REF_LIB.exists():
            if not REFERENCE_SRC.exists():
                return None
            subprocess.run(["make", "-C", str(ODIR), "-j8", "ref"], check=True,
                           capture_output=True)
        import importlib.util
        spec = importlib.util.spec_from_file_location("oracle_reference", __file__)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        mod.LIB = REF_LIB
        mod.BACKEND = "reference"
        mod._REF_MODULE = mod
        _REF_MODULE = mod
    return _REF_MODULE

OK, INVALID_ARGUMENT, DOMAIN_ERROR, NO_SUPPORTED_CENTERS, RUNTIME_ERROR = 0, 1, 2, 3, 4
UNSUPPORTED = 9


class OracleError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


class KP(C.Structure):
    _fields_ = [("sigma", C.c_double), ("sigma_eps", C.c_double), ("lambda_", C.c_double),
                ("cutoff_radius", C.c_double)]


class CP(C.Structure):
    _fields_ = [("mesh_resolution", C.c_double), ("accept_radius", C.c_double),
                ("accept_count", C.c_int), ("pad", C.c_int), ("roi_min_x", C.c_double),
                ("roi_min_y", C.c_double), ("roi_max_x", C.c_double), ("roi_max_y", C.c_double)]


_lib = None


def load():
    global _lib
    if _lib is None:
        if not LIB.exists() and BACKEND == "port":
            subprocess.run(["make", "-C", str(ODIR)], check=True, capture_output=True)
        _lib = C.CDLL(str(LIB))
        _lib.orc_last_error.restype = C.c_char_p
        _lib.orc_rng_new.restype = C.c_void_p
        _lib.orc_rng_new.argtypes = [C.c_ulonglong]
        _lib.orc_normal_new.restype = C.c_void_p
        _lib.orc_normal_new.argtypes = [C.c_double, C.c_double]
        for f in ("orc_rng_free", "orc_normal_free", "orc_model_free", "orc_grid_free"):
            getattr(_lib, f).argtypes = [C.c_void_p]
        _lib.orc_uniform.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_size_t, C.c_void_p]
        _lib.orc_uniform_int.argtypes = [C.c_void_p, C.c_int, C.c_int]
        _lib.orc_normal.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
        _lib.orc_grid_new.restype = C.c_void_p
        _lib.orc_grid_new.argtypes = [C.c_double, C.c_void_p, C.c_void_p, C.c_size_t]
        _lib.orc_grid_query.restype = C.c_size_t
        _lib.orc_grid_query.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double,
                                        C.c_void_p, C.c_size_t]
        _lib.orc_sigma_tilde.restype = C.c_double
        _lib.orc_moment_scale.restype = C.c_double
        for f in ("orc_model_num_centers", "orc_model_num_blocks", "orc_model_block_size",
                  "orc_model_centers_near"):
            getattr(_lib, f).restype = C.c_size_t
        _lib.orc_model_num_centers.argtypes = [C.c_void_p]
        _lib.orc_model_num_blocks.argtypes = [C.c_void_p]
        _lib.orc_model_block_size.argtypes = [C.c_void_p, C.c_uint]
        _lib.orc_model_centers_near.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_void_p,
                                                C.c_size_t]
        for f in ("orc_model_weights", "orc_model_set_weights", "orc_model_block_index",
                  "orc_model_kernel"):
            getattr(_lib, f).argtypes = [C.c_void_p, C.c_void_p]
        _lib.orc_model_centers.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_model_block_members.argtypes = [C.c_void_p, C.c_uint, C.c_void_p]
        _lib.orc_model_block_info_inverse.argtypes = [C.c_void_p, C.c_uint, C.c_void_p]
        _lib.orc_model_predict.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        _lib.orc_model_moment_feature.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_void_p,
                                                  C.c_void_p, C.c_size_t, C.c_void_p]
        _lib.orc_model_recursive_update.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p,
                                                    C.c_void_p, C.c_size_t, C.c_size_t, C.c_int,
                                                    C.c_void_p]
        _lib.orc_model_new.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                       C.c_void_p]
        _lib.orc_fit_batch_ridge.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                             C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p,
                                             C.c_size_t, C.c_void_p]
        _lib.orc_model_save.argtypes = [C.c_void_p, C.c_char_p]
        _lib.orc_model_load.argtypes = [C.c_char_p, C.c_void_p]
        _lib.orc_supported_mesh_nodes.argtypes = [
            C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, C.c_double, C.c_double,
            C.c_double, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_void_p,
            C.c_void_p, C.c_size_t, C.c_void_p]
        _lib.orc_kernel_eval.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double,
                                         C.c_double, C.c_double, C.c_void_p]
        _lib.orc_manifold_rows.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_size_t, C.c_double,
                                           C.c_double, C.c_double, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        _lib.orc_lm_step.argtypes = [C.c_void_p, C.c_double, C.c_void_p]
        _lib.orc_so3_exp.argtypes = [C.c_void_p, C.c_void_p]
        _lib.orc_select_ground_points.argtypes = [
            C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p,
            C.c_void_p, C.c_double, C.c_double, C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p,
            C.c_void_p]
        _lib.orc_terrain_error_histogram.argtypes = [
            C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_double, C.c_int,
            C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_map_new.restype = C.c_void_p
        _lib.orc_map_new.argtypes = [C.c_double, C.c_size_t]
        _lib.orc_map_free.argtypes = [C.c_void_p]
        _lib.orc_map_insert.argtypes = [C.c_void_p] + [C.c_void_p] * 5 + [C.c_size_t, C.c_void_p,
                                                                          C.c_void_p]
        _lib.orc_map_points.restype = C.c_size_t
        _lib.orc_map_points.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_size_t]
        _lib.orc_knn.restype = C.c_size_t
        _lib.orc_knn.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                                 C.c_double, C.c_void_p, C.c_int]
        _lib.orc_build_correspondences.restype = C.c_size_t
        _lib.orc_build_correspondences.argtypes = [C.c_void_p] + [C.c_void_p] * 4 + [
            C.c_size_t] + [C.c_void_p] * 10
        _lib.orc_feature_normal_eq.argtypes = [C.c_size_t] + [C.c_void_p] * 7
        _lib.orc_export_grid.restype = C.c_size_t
        _lib.orc_export_grid.argtypes = [C.c_void_p, C.c_double, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_size_t]
    return _lib


def _chk(st):
    if st != OK:
        raise OracleError(st, load().orc_last_error().decode())


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


# ---- RNG (std::mt19937_64 + libstdc++ distributions) ------------------------
class Rng:
    def __init__(self, seed: int):
        self.h = load().orc_rng_new(seed)

    def uniform(self, lo, hi, n=None):
        k = 1 if n is None else n
        out = np.empty(k)
        load().orc_uniform(self.h, lo, hi, k, _p(out))
        return float(out[0]) if n is None else out

    def uniform_int(self, lo, hi):
        return load().orc_uniform_int(self.h, lo, hi)

    def __del__(self):
        try:
            load().orc_rng_free(self.h)
        except Exception:
            pass


class Normal:
    def __init__(self, mean=0.0, sd=1.0):
        self.h = load().orc_normal_new(mean, sd)

    def draw(self, rng: Rng, n=None):
        k = 1 if n is None else n
        out = np.empty(k)
        load().orc_normal(self.h, rng.h, k, _p(out))
        return float(out[0]) if n is None else out

    def __del__(self):
        try:
            load().orc_normal_free(self.h)
        except Exception:
            pass


def kp(kernel) -> KP:
    return KP(kernel.sigma, kernel.sigma_eps, kernel.lambda_, kernel.cutoff_radius)


def cp(centers) -> CP:
    r = centers.roi
    return CP(centers.mesh_resolution, centers.accept_radius, int(centers.accept_count), 0,
              r.min[0], r.min[1], r.max[0], r.max[1])


def kernel_finalize(kernel):
    k = kp(kernel)
    _chk(load().orc_kernel_finalize(C.byref(k)))
    return k.cutoff_radius


def kernel_eval(kernel, x, c, bw):
    out = C.c_double()
    _chk(load().orc_kernel_eval(C.byref(kp(kernel)), x[0], x[1], c[0], c[1], bw, C.byref(out)))
    return out.value


def sigma_tilde(kernel):
    return load().orc_sigma_tilde(C.byref(kp(kernel)))


def moment_scale(kernel):
    return load().orc_moment_scale(C.byref(kp(kernel)))


class Grid:
    def __init__(self, cell, pts):
        p = _f64(pts).reshape(-1, 2)
        x, y = _f64(p[:, 0]), _f64(p[:, 1])
        self.h = load().orc_grid_new(cell, _p(x), _p(y), len(x))

    def radius_query(self, q, r):
        out = np.empty(1 << 16, dtype=np.uint32)
        n = load().orc_grid_query(self.h, q[0], q[1], r, _p(out), len(out))
        return out[:n].copy()

    def __del__(self):
        try:
            load().orc_grid_free(self.h)
        except Exception:
            pass


def supported_mesh_nodes(xy, z, roi, res, r_a, count, throw_empty=False):
    p = _f64(xy).reshape(-1, 2)
    x, y, zz = _f64(p[:, 0]), _f64(p[:, 1]), _f64(z).reshape(-1)
    cap = max(1024, 4 * len(x) + 1024)
    ox, oy = np.empty(cap), np.empty(cap)
    n = C.c_size_t()
    _chk(load().orc_supported_mesh_nodes(_p(x), _p(y), _p(zz), len(x), len(zz), roi.min[0],
                                         roi.min[1], roi.max[0], roi.max[1], res, r_a, count,
                                         1 if throw_empty else 0, _p(ox), _p(oy), cap,
                                         C.byref(n)))
    return np.stack([ox[: n.value], oy[: n.value]], 1)


class Model:
    def __init__(self, kernel=None, centers=None, _h=None):
        if _h is not None:
            self.h = _h
            return
        c = _f64(centers.centers).reshape(-1, 2)
        cx, cy = _f64(c[:, 0]), _f64(c[:, 1])
        h = C.c_void_p()
        _chk(load().orc_model_new(C.byref(kp(kernel)), C.byref(cp(centers)), _p(cx), _p(cy),
                                  len(cx), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            load().orc_model_free(self.h)
        except Exception:
            pass

    def num_centers(self):
        return load().orc_model_num_centers(self.h)

    def num_blocks(self):
        return load().orc_model_num_blocks(self.h)

    def kernel_cutoff(self):
        k = KP()
        load().orc_model_kernel(self.h, C.byref(k))
        return k.cutoff_radius

    def centers(self):
        n = self.num_centers()
        cx, cy = np.empty(n), np.empty(n)
        load().orc_model_centers(self.h, _p(cx), _p(cy))
        return np.stack([cx, cy], 1)

    def weights(self):
        w = np.empty(self.num_centers())
        load().orc_model_weights(self.h, _p(w))
        return w

    def set_weights(self, w):
        w = _f64(w)
        load().orc_model_set_weights(self.h, _p(w))

    def block_index(self):
        out = np.empty(self.num_centers(), dtype=np.uint32)
        load().orc_model_block_index(self.h, _p(out))
        return out

    def block_members(self, b):
        n = load().orc_model_block_size(self.h, b)
        out = np.empty(n, dtype=np.uint32)
        load().orc_model_block_members(self.h, b, _p(out))
        return out

    def set_block_info_inverse(self, b, a):
        """Reference backend only (snapshot round trip)."""
        a = np.asfortranarray(np.asarray(a, dtype=np.float64))
        f = load().orc_model_set_block_info_inverse
        f.argtypes = [C.c_void_p, C.c_uint, C.c_void_p]
        _chk(f(self.h, int(b), a.ctypes.data_as(C.c_void_p)))

    def block_info_inverse(self, b):
        n = load().orc_model_block_size(self.h, b)
        out = np.empty(n * n)
        load().orc_model_block_info_inverse(self.h, b, _p(out))
        return out.reshape(n, n, order="F")

    def predict(self, xy, threads=1):
        p = _f64(xy).reshape(-1, 2)
        x, y = _f64(p[:, 0]), _f64(p[:, 1])
        n = len(x)
        z, s, gx, gy = np.empty(n), np.empty(n, dtype=np.uint8), np.empty(n), np.empty(n)
        _chk(load().orc_model_predict(self.h, _p(x), _p(y), n, _p(z), _p(s), _p(gx), _p(gy),
                                      threads))
        return z, s, gx, gy

    def scales(self, xy, threads=None):
        """Parity scales per point: (sum |w kappa|, sum |w kappa| d / s^2)."""
        import os
        p = _f64(xy).reshape(-1, 2)
        x, y = _f64(p[:, 0]), _f64(p[:, 1])
        s, g = np.empty(len(x)), np.empty(len(x))
        f = load().orc_model_scales
        f.argtypes = [C.c_void_p] + [C.c_void_p] * 2 + [C.c_size_t] + [C.c_void_p] * 2 + [C.c_int]
        _chk(f(self.h, _p(x), _p(y), len(x), _p(s), _p(g), int(threads or os.cpu_count() or 1)))
        return s, g

    def centers_near(self, q):
        out = np.empty(1 << 16, dtype=np.uint32)
        n = load().orc_model_centers_near(self.h, q[0], q[1], _p(out), len(out))
        return out[:n].copy()

    def moment_feature(self, q):
        ids, vals = np.empty(1 << 16, dtype=np.uint32), np.empty(1 << 16)
        n = C.c_size_t()
        _chk(load().orc_model_moment_feature(self.h, q[0], q[1], _p(ids), _p(vals), len(ids),
                                             C.byref(n)))
        return ids[: n.value].copy(), vals[: n.value].copy()

    def recursive_update(self, xy, z, allow_birth=True):
        p = _f64(xy).reshape(-1, 2)
        x, y, zz = _f64(p[:, 0]), _f64(p[:, 1]), _f64(z).reshape(-1)
        rep = (C.c_ulonglong * 4)()
        _chk(load().orc_model_recursive_update(self.h, _p(x), _p(y), _p(zz), len(x), len(zz),
                                               1 if allow_birth else 0, rep))
        return dict(active_blocks=rep[0], active_centers=rep[1], born_centers=rep[2],
                    rejected=bool(rep[3]))

    def save(self, path):
        _chk(load().orc_model_save(self.h, str(path).encode()))

    @staticmethod
    def load_file(path):
        h = C.c_void_p()
        _chk(load().orc_model_load(str(path).encode(), C.byref(h)))
        return Model(_h=h)

    def error_histogram(self, xy, z, trim_fraction=0.0, bins=25):
        """metrics.cpp:199-232 restated: dict(edges, counts, trimmed, overflow)."""
        xy = _f64(xy)
        z = _f64(z)
        x, y = np.ascontiguousarray(xy[:, 0]), np.ascontiguousarray(xy[:, 1])
        edges = np.empty(bins + 1)
        counts = np.zeros(bins, dtype=np.uint64)
        tr, ov = C.c_ulonglong(), C.c_ulonglong()
        _chk(load().orc_terrain_error_histogram(self.h, _p(x), _p(y), _p(z), len(z),
                                                float(trim_fraction), int(bins), _p(edges),
                                                _p(counts), C.byref(tr), C.byref(ov)))
        return {"edges": edges, "counts": counts, "trimmed": tr.value, "overflow": ov.value}

    def export_grid(self, grid_step):
        """terrain_model.cpp:255-267 restated: supported grid points and heights."""
        cap = 1 << 22
        x, y, z = np.empty(cap), np.empty(cap), np.empty(cap)
        n = load().orc_export_grid(self.h, float(grid_step), _p(x), _p(y), _p(z), cap)
        assert n <= cap
        return x[:n].copy(), y[:n].copy(), z[:n].copy()

    def manifold_rows(self, R, t, h, wheel_radius=0.0, lambda_M=1.0, huber=0.05, threads=1):
        Rm, tv = _f64(R).reshape(9), _f64(t).reshape(3)
        ha = _f64(h).reshape(-1, 3)
        hx, hy, hz = _f64(ha[:, 0]), _f64(ha[:, 1]), _f64(ha[:, 2])
        n = len(hx)
        r, J, v, raw, ne = (np.empty(n), np.empty(6 * n), np.empty(n, dtype=np.uint8),
                            np.empty(n), np.empty(29))
        _chk(load().orc_manifold_rows(self.h, _p(Rm), _p(tv), _p(hx), _p(hy), _p(hz), n,
                                      wheel_radius, lambda_M, huber, _p(r), _p(J), _p(v), _p(raw),
                                      _p(ne), threads))
        return dict(r=r, J=J.reshape(n, 6), valid=v, raw=raw), ne


def select_ground_points(p, kind, R, t, roi, radius, voxel, max_points):
    """pipeline.cpp:150-170 restated (oracle)."""
    p = np.ascontiguousarray(np.asarray(p, dtype=np.float64))
    px, py, pz = (np.ascontiguousarray(p[:, j]) for j in range(3))
    kind = np.ascontiguousarray(np.asarray(kind, dtype=np.uint8))
    Rm = np.ascontiguousarray(np.asarray(R, dtype=np.float64).reshape(9))
    tv = np.ascontiguousarray(np.asarray(t, dtype=np.float64).reshape(3))
    r4 = np.array([roi.min[0], roi.min[1], roi.max[0], roi.max[1]], dtype=np.float64)
    cap = max(int(max_points), 1)
    ox, oy, oz = np.empty(cap), np.empty(cap), np.empty(cap)
    n = C.c_size_t()
    _chk(load().orc_select_ground_points(_p(px), _p(py), _p(pz), _p(kind), len(kind), _p(Rm),
                                         _p(tv), _p(r4), float(radius), float(voxel),
                                         int(max_points), _p(ox), _p(oy), _p(oz), C.byref(n)))
    k = n.value
    return np.stack([ox[:k], oy[:k]], 1), oz[:k].copy()


MATCH_DEFAULTS = dict(corr_gate=1.0, huber_delta=0.1, plane_fit_tol=0.025, plane_eig_ratio=5.0,
                      edge_eig_ratio=3.0, edge_fit_tol=0.05, edge_min_extent=0.05,
                      trim_ratio=5.0, trim_floor=0.003, ground_corr_voxel=0.25,
                      ground_corr_radius=4.0)


def _cfg_vec(cfg):
    c = dict(MATCH_DEFAULTS)
    c.update(cfg or {})
    return np.array([c[k] for k in MATCH_DEFAULTS], dtype=np.float64)


class LocalMap:
    """local_map.cpp restated (oracle)."""

    def __init__(self, voxel_size=0.1, window=20):
        self.h = load().orc_map_new(float(voxel_size), int(window))

    def __del__(self):
        try:
            load().orc_map_free(self.h)
        except Exception:
            pass

    def insert(self, p, kind, label, R, t):
        p = _f64(p)
        cols = [np.ascontiguousarray(p[:, j]) for j in range(3)]
        kind = np.ascontiguousarray(np.asarray(kind, dtype=np.uint8))
        label = np.ascontiguousarray(np.asarray(label, dtype=np.int32))
        load().orc_map_insert(self.h, _p(cols[0]), _p(cols[1]), _p(cols[2]), _p(kind), _p(label),
                              len(kind), _p(_f64(R).reshape(9)), _p(_f64(t).reshape(3)))

    def points(self, kind):
        n = load().orc_map_points(self.h, kind, None, None, 0)
        xyz = np.empty((n, 3))
        lab = np.empty(n, dtype=np.int32)
        load().orc_map_points(self.h, kind, _p(xyz), _p(lab), n)
        return xyz, lab

    def knn(self, kind, q, k, gate, tree=True):
        out = np.empty(k, dtype=np.uint32)
        m = load().orc_knn(self.h, kind, float(q[0]), float(q[1]), float(q[2]), int(k),
                           float(gate), _p(out), int(bool(tree)))
        return out[:m].copy()

    def build_correspondences(self, p, kind, R, t, cfg=None):
        p = _f64(p)
        cols = [np.ascontiguousarray(p[:, j]) for j in range(3)]
        kind = np.ascontiguousarray(np.asarray(kind, dtype=np.uint8))
        n = len(kind)
        ck = np.empty(n, dtype=np.int32)
        cf = np.empty(n, dtype=np.uint32)
        prm = np.empty((n, 7))
        w = np.empty(n)
        lab = np.empty(n, dtype=np.int32)
        dist = np.empty(n)
        fq = np.empty(n)
        m = load().orc_build_correspondences(
            self.h, _p(cols[0]), _p(cols[1]), _p(cols[2]), _p(kind), n, _p(_f64(R).reshape(9)),
            _p(_f64(t).reshape(3)), _p(_cfg_vec(cfg)), _p(ck), _p(cf), _p(prm), _p(w), _p(lab),
            _p(dist), _p(fq))
        return {"kind": ck[:m].copy(), "feature": cf[:m].copy(), "params": prm[:m].copy(),
                "weight": w[:m].copy(), "label": lab[:m].copy(), "dist": dist[:m].copy(),
                "fitq": fq[:m].copy()}


def feature_normal_eq(corr, p_sensor, R, t):
    """Feature rows of total_cost (scan_matcher.cpp:185-216) -> ne29."""
    ck = np.ascontiguousarray(corr["kind"], dtype=np.int32)
    ps = _f64(np.asarray(p_sensor)[corr["feature"]])
    prm = _f64(corr["params"])
    w = _f64(corr["weight"])
    out = np.empty(29)
    load().orc_feature_normal_eq(len(ck), _p(ck), _p(ps), _p(prm), _p(w), _p(_f64(R).reshape(9)),
                                 _p(_f64(t).reshape(3)), _p(out))
    return out


def fit_batch_ridge(kernel, centers, xy, z):
    c = _f64(centers.centers).reshape(-1, 2)
    cx, cy = _f64(c[:, 0]), _f64(c[:, 1])
    p = _f64(xy).reshape(-1, 2)
    x, y, zz = _f64(p[:, 0]), _f64(p[:, 1]), _f64(z).reshape(-1)
    h = C.c_void_p()
    _chk(load().orc_fit_batch_ridge(C.byref(kp(kernel)), C.byref(cp(centers)), _p(cx), _p(cy),
                                    len(cx), _p(x), _p(y), _p(zz), len(x), C.byref(h)))
    return Model(_h=h)


def lm_step(ne29, mu):
    d = np.empty(6)
    ne = _f64(ne29)
    st = load().orc_lm_step(_p(ne), mu, _p(d))
    return d, st == OK


def so3_exp(w):
    R = np.empty(9)
    load().orc_so3_exp(_p(_f64(w)), _p(R))
    return R.reshape(3, 3)


# ---- reference-only: simulator bundles, lm_solve, the odometry loop ----------
def _ref_fn(name, restype, argtypes):
    f = getattr(load(), name)
    f.restype = restype
    f.argtypes = argtypes
    return f


class SimBundle:
    """sim::simulate(stock_scene(scene), seed) (sensors.cpp:249-271) with an
    optional azimuth x elevation ray override, first `max_scans` scans."""

    def __init__(self, scene="staircase", seed=11, az=0, el=0, max_scans=0):
        f = _ref_fn("ref_sim_new", C.c_void_p, [C.c_char_p, C.c_ulonglong, C.c_int, C.c_int, C.c_long])
        self.h = f(scene.encode(), int(seed), int(az), int(el), int(max_scans))
        if not self.h:
            raise OracleError(RUNTIME_ERROR, load().orc_last_error().decode())

    def __del__(self):
        try:
            _ref_fn("ref_sim_free", None, [C.c_void_p])(self.h)
        except Exception:
            pass

    def num_scans(self):
        return _ref_fn("ref_sim_num_scans", C.c_size_t, [C.c_void_p])(self.h)

    def scan(self, k):
        f = _ref_fn("ref_sim_scan", C.c_size_t, [C.c_void_p, C.c_size_t] + [C.c_void_p] * 5 + [C.c_size_t])
        n = f(self.h, k, None, None, None, None, None, 0)
        px, py, pz = np.empty(n), np.empty(n), np.empty(n)
        kind, lab = np.empty(n, dtype=np.uint8), np.empty(n, dtype=np.int32)
        f(self.h, k, _p(px), _p(py), _p(pz), _p(kind), _p(lab), n)
        return np.stack([px, py, pz], 1), kind, lab

    def gt(self, k):
        R, t, ts = np.empty(9), np.empty(3), C.c_double()
        _ref_fn("ref_sim_gt", None, [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p])(
            self.h, k, _p(R), _p(t), C.byref(ts))
        return R.reshape(3, 3), t, ts.value

    def roi(self):
        r = np.empty(4)
        _ref_fn("ref_sim_roi", None, [C.c_void_p, C.c_void_p])(self.h, _p(r))
        return r

    def wheel_radius(self):
        return _ref_fn("ref_sim_wheel_radius", C.c_double, [C.c_void_p])(self.h)

    def wheel_arms(self, t):
        hL, hR = np.empty(3), np.empty(3)
        ok = _ref_fn("ref_sim_wheel_arms", C.c_int, [C.c_void_p, C.c_double, C.c_void_p, C.c_void_p])(
            self.h, float(t), _p(hL), _p(hR))
        return (hL, hR) if ok else None


def run_config_json(**kw):
    """RunConfig JSON (pipeline.cpp:22-89); nested dicts for kernel/solver/map."""
    import json
    return json.dumps(kw)


def odometry(bundle: SimBundle, config_json: str, mode=0):
    """The reference odometry loop over a bundle (mode 1: pipeline::run_odometry
    itself; mode 0: the same loop restated from its public pieces, also
    recording predicted poses and the lever arms each lm_solve saw)."""
    n = bundle.num_scans()
    poses, preds, arms = np.zeros((n, 12)), np.zeros((n, 12)), np.zeros((n, 7))
    ints, terr, dbl = np.zeros((n, 8), dtype=np.int32), np.zeros((n, 4)), np.zeros((n, 3))
    f = _ref_fn("ref_odometry", C.c_int, [C.c_void_p, C.c_char_p, C.c_int] + [C.c_void_p] * 6)
    _chk(f(bundle.h, config_json.encode(), int(mode), _p(poses), _p(preds), _p(arms), _p(ints), _p(terr),
           _p(dbl)))
    keys = ("held", "inserted", "converged", "failed", "degenerate", "outer_iterations",
            "accepted_steps", "correspondences")
    out = {k: ints[:, i].copy() for i, k in enumerate(keys)}
    out.update(R=poses[:, :9].reshape(n, 3, 3), t=poses[:, 9:].copy(),
               R_pred=preds[:, :9].reshape(n, 3, 3), t_pred=preds[:, 9:].copy(),
               hL=arms[:, :3].copy(), hR=arms[:, 3:6].copy(), has_arms=arms[:, 6] > 0,
               active_blocks=terr[:, 0].astype(int), active_centers=terr[:, 1].astype(int),
               born_centers=terr[:, 2].astype(int), rejected=terr[:, 3] > 0,
               final_cost=dbl[:, 0].copy(), wall_ms=dbl[:, 1].copy(), min_eig=dbl[:, 2].copy())
    return out


def lm_solve(local_map, P, kind, R0, t0, model=None, hL=None, hR=None, wheel_radius=0.0, cfg=None,
             lambda_M=1.0, manifold_huber=0.05):
    """match::lm_solve on the reference (scan_matcher.cpp:257-358)."""
    P = _f64(P)
    cols = [np.ascontiguousarray(P[:, j]) for j in range(3)]
    kind = np.ascontiguousarray(np.asarray(kind, dtype=np.uint8))
    R, t, rep, trace = np.empty(9), np.empty(3), np.empty(8), np.empty(256)
    nt = C.c_size_t()
    f = _ref_fn("ref_lm_solve", C.c_int,
                [C.c_void_p] * 5 + [C.c_size_t] + [C.c_void_p] * 5 + [C.c_double, C.c_void_p, C.c_double,
                                                                   C.c_double] + [C.c_void_p] * 4 +
                [C.c_size_t, C.c_void_p])
    _chk(f(local_map.h, _p(cols[0]), _p(cols[1]), _p(cols[2]), _p(kind), len(kind),
           _p(_f64(R0).reshape(9)), _p(_f64(t0).reshape(3)), model.h if model is not None else None,
           None if hL is None else _p(_f64(hL)), None if hR is None else _p(_f64(hR)), float(wheel_radius),
           _p(_cfg_vec(cfg)), float(lambda_M), float(manifold_huber), _p(R), _p(t), _p(rep), _p(trace),
           len(trace), C.byref(nt)))
    keys = ("converged", "failed", "degenerate", "outer_iterations", "accepted_steps",
            "correspondence_count", "final_cost", "smallest_feature_eigenvalue")
    r = dict(zip(keys, rep.tolist()))
    for k in ("converged", "failed", "degenerate"):
        r[k] = bool(r[k])
    for k in ("outer_iterations", "accepted_steps", "correspondence_count"):
        r[k] = int(r[k])
    r["cost_trace"] = trace[: min(nt.value, len(trace))].copy()
    return R.reshape(3, 3), t, r
