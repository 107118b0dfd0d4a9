// Feature correspondences on the device:
//   LocalMap::insert / rebuild (local_map.cpp:19-60): pose transform, first
//     point per (kind, voxel) in scan order, sliding window of frames;
//   KdTree3::knn (kdtree.hpp:31-99): exact k nearest within the gate,
//     closest first, ties by id — here a uniform grid (cell > gate, so the
//     3x3x3 neighbourhood is complete) and a per-query sorted top-k;
//   build_correspondences (scan_matcher.cpp:44-183): ground thinning, kNN,
//     centroid / scatter in neighbour order, 3x3 symmetric eigen sweeps,
//     line / plane gates, adaptive trims (exact order statistics by sort);
//   total_cost feature rows (scan_matcher.cpp:185-216, residuals.cpp:7-25)
//     reduced to J^T J, J^T r, cost.
// Built with -fmad=false: the scalar geometry rounds like the oracle's
// restatement (the reference's Eigen eigen solver itself is unpinned).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cmath>
#include <deque>
#include <vector>

#include "internal.cuh"

struct tlg_map {
  tlg_ctx* ctx = nullptr;
  double voxel = 0.1;
  size_t window = 20;
  struct Frame {
    tlg::DBuf<double> pts[2];  // xyz per point, [0] edge, [1] planar
    tlg::DBuf<int> lab[2];
    size_t n[2] = {0, 0};
  };
  std::deque<Frame> frames;
  tlg::DBuf<double> pts[2];
  tlg::DBuf<int> lab[2];
  size_t n[2] = {0, 0};
  struct Grid {
    tlg::DBuf<int> start;      // dims + 1
    tlg::DBuf<uint32_t> ids;   // point ids sorted by cell (stable: ascending within a cell)
    double org[3] = {0, 0, 0};
    double cell = 0.0;
    int dim[3] = {0, 0, 0};
    double gate = -1.0;
  } grid[2];
  // last correspondences (device, feature order after trims)
  tlg::DBuf<int> c_kind;
  tlg::DBuf<uint32_t> c_feat;
  tlg::DBuf<double> c_par, c_w, c_dist, c_q, c_ps;
  tlg::DBuf<int> c_lab;
  size_t nc = 0;
};

namespace tlg {
namespace {

struct Pose {
  double R[9];
  double t[3];
};

__device__ __forceinline__ void xform(const Pose& P, double f0, double f1, double f2, double& x,
                                      double& y, double& z) {
  x = ((P.R[0] * f0 + P.R[1] * f1) + P.R[2] * f2) + P.t[0];
  y = ((P.R[3] * f0 + P.R[4] * f1) + P.R[5] * f2) + P.t[1];
  z = ((P.R[6] * f0 + P.R[7] * f1) + P.R[8] * f2) + P.t[2];
}

// local_map.cpp:10-16
__device__ __forceinline__ uint64_t map_voxel_key(double x, double y, double z, double size) {
  auto q = [&](double v) {
    return static_cast<uint64_t>(static_cast<int64_t>(floor(v / size)) & 0x1fffff);
  };
  return (q(x) << 42) | (q(y) << 21) | q(z);
}

__global__ void k_map_keys(const double* __restrict__ px, const double* __restrict__ py,
                           const double* __restrict__ pz, const uint8_t* __restrict__ kind,
                           size_t n, Pose P, double voxel, double* __restrict__ xyz,
                           uint64_t* __restrict__ keys, uint32_t* __restrict__ idx) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x, y, z;
  xform(P, px[i], py[i], pz[i], x, y, z);
  xyz[3 * i] = x;
  xyz[3 * i + 1] = y;
  xyz[3 * i + 2] = z;
  const uint64_t cls = kind[i] == 0 ? 0ull : 1ull;  // edge / planar (ground kept as planar)
  const uint64_t key = voxel > 0.0 ? map_voxel_key(x, y, z, voxel) : static_cast<uint64_t>(i);
  keys[i] = (cls << 63) | key;
  idx[i] = static_cast<uint32_t>(i);
}

// run heads of sorted keys; with `sentinel`, the key ~0 marks excluded entries
__global__ void k_first_of_run(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx,
                               size_t n, int sentinel, uint8_t* __restrict__ first) {
  const size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint64_t k = keys[p];
  if ((!sentinel || k != ~0ull) && (p == 0 || keys[p - 1] != k)) first[idx[p]] = 1;
}

__global__ void k_flag_class(const uint8_t* __restrict__ first, const uint8_t* __restrict__ kind,
                             size_t n, int cls, uint8_t* __restrict__ out) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = first[i] && ((kind[i] == 0 ? 0 : 1) == cls);
}

__global__ void k_gather_pts(const uint32_t* __restrict__ sel, size_t cnt,
                             const double* __restrict__ xyz, const int* __restrict__ label,
                             double* __restrict__ out, int* __restrict__ out_lab) {
  const size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (j >= cnt) return;
  const uint32_t i = sel[j];
  out[3 * j] = xyz[3 * i];
  out[3 * j + 1] = xyz[3 * i + 1];
  out[3 * j + 2] = xyz[3 * i + 2];
  out_lab[j] = label ? label[i] : -1;
}

struct GridView3 {
  const double* pts;
  const int* start;
  const uint32_t* ids;
  double org[3];
  double cell;
  int dim[3];
};

__global__ void k_cell_keys(const double* __restrict__ pts, size_t n, GridView3 g,
                            uint32_t* __restrict__ keys, uint32_t* __restrict__ idx) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c[3];
  for (int a = 0; a < 3; ++a)
    c[a] = min(max(static_cast<int>(floor((pts[3 * i + a] - g.org[a]) / g.cell)), 0), g.dim[a] - 1);
  keys[i] = static_cast<uint32_t>((c[2] * g.dim[1] + c[1]) * g.dim[0] + c[0]);
  idx[i] = static_cast<uint32_t>(i);
}

__global__ void k_cell_count(const uint32_t* __restrict__ keys, size_t n, int* __restrict__ cnt) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&cnt[keys[i]], 1);
}

// kdtree.hpp semantics: the k smallest (d2, id) with d2 <= gate^2,
// d2 = (p - q).squaredNorm(); returns the count found. Cells are visited in
// shells of growing Chebyshev radius r around q's cell; a point first seen in
// shell r is at least (r - 2) cells away even allowing one cell of index
// rounding, so the search stops once ((r - 2) c)^2 exceeds the current k-th
// distance (or the gate) — the result equals the exhaustive search's.
// Run by a group of G lanes (one query per group): each lane scans a
// stride-G share of every visited cell into its own top-K, and after each
// shell the group merges the lanes' lists (K rounds of a lexicographic
// (d2, id) minimum over the group; a point reaches the lists of one lane only,
// but after a merge every lane continues from the merged list, so equal
// entries are advanced together). The stopping test runs on the merged list
// before each shell: the result is the sequential search's.
template <int K, int G>
__device__ int knn_group(const GridView3& g, double qx, double qy, double qz, double gate2,
                         int glane, unsigned gmask, uint32_t (&ids)[K], double (&d2s)[K]) {
  int m = 0;  // entries in this lane's list
  int c[3];
  const double q[3] = {qx, qy, qz};
  for (int a = 0; a < 3; ++a) c[a] = static_cast<int>(floor((q[a] - g.org[a]) / g.cell));
  auto insert = [&](uint32_t id, double d2) {
    if (!(d2 <= gate2)) return;
    if (m == K && !(d2 < d2s[K - 1] || (d2 == d2s[K - 1] && id < ids[K - 1]))) return;
    int j = m < K ? m++ : K - 1;
    while (j > 0 && (d2s[j - 1] > d2 || (d2s[j - 1] == d2 && ids[j - 1] > id))) {
      d2s[j] = d2s[j - 1];
      ids[j] = ids[j - 1];
      --j;
    }
    d2s[j] = d2;
    ids[j] = id;
  };
  auto visit = [&](int cx, int cy, int cz) {
    if (cx < 0 || cx >= g.dim[0] || cy < 0 || cy >= g.dim[1] || cz < 0 || cz >= g.dim[2]) return;
    const int cell = (cz * g.dim[1] + cy) * g.dim[0] + cx;
    for (int s = g.start[cell] + glane; s < g.start[cell + 1]; s += G) {
      const uint32_t id = g.ids[s];
      const double ex = g.pts[3 * id] - qx, ey = g.pts[3 * id + 1] - qy, ez = g.pts[3 * id + 2] - qz;
      insert(id, (ex * ex + ey * ey) + ez * ez);
    }
  };
  auto merge = [&]() {
    uint32_t mi[K];
    double md[K];
    int p = 0, mm = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double cd = INFINITY;
      uint32_t ci = 0xffffffffu;
#pragma unroll
      for (int t = 0; t < K; ++t)
        if (t == p && p < m) {
          cd = d2s[t];
          ci = ids[t];
        }
      double bd = cd;
      uint32_t bi = ci;
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) {
        const double od = __shfl_xor_sync(gmask, bd, o, G);
        const uint32_t oi = __shfl_xor_sync(gmask, bi, o, G);
        if (od < bd || (od == bd && oi < bi)) {
          bd = od;
          bi = oi;
        }
      }
      md[k] = bd;
      mi[k] = bi;
      if (bi != 0xffffffffu) mm = k + 1;
      if (ci == bi && cd == bd && p < m) ++p;
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      d2s[k] = md[k];
      ids[k] = mi[k];
    }
    m = mm;
  };
  const int rmax = max(max(g.dim[0], g.dim[1]), g.dim[2]);
  const double eps = 1e-9 * (fabs(g.org[0]) + fabs(g.org[1]) + fabs(g.org[2]) + g.cell * rmax);
  for (int r = 0; r <= rmax; ++r) {
    if (r >= 1) {
      merge();
      double lb = INFINITY;
      for (int a = 0; a < 3; ++a) {
        const double hi_face = g.org[a] + (c[a] + r) * g.cell - q[a];
        const double lo_face = q[a] - (g.org[a] + (c[a] - r + 1) * g.cell);
        lb = fmin(lb, fmin(hi_face, lo_face));
      }
      lb -= eps;
      if (lb > 0.0) {
        const double lb2 = lb * lb;
        if (lb2 > gate2) break;
        if (m == K && lb2 > d2s[K - 1]) break;
      }
    }
    for (int dz = -r; dz <= r; ++dz)
      for (int dy = -r; dy <= r; ++dy) {
        const bool face = (dz == -r || dz == r || dy == -r || dy == r);
        if (face) {
          for (int dx = -r; dx <= r; ++dx) visit(c[0] + dx, c[1] + dy, c[2] + dz);
        } else {
          visit(c[0] - r, c[1] + dy, c[2] + dz);
          if (r > 0) visit(c[0] + r, c[1] + dy, c[2] + dz);
        }
      }
    if (r == rmax) merge();
  }
  return m;
}

// cyclic Jacobi, identical to the oracle's eigen_sym3 (row-major in,
// ascending eigenvalues, column-major vectors)
__device__ void eigen_sym3(const double A[9], double ev[3], double V[9]) {
  double a[3][3], v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) a[i][j] = A[3 * i + j];
  for (int sweep = 0; sweep < 60; ++sweep) {
    const double off = fabs(a[0][1]) + fabs(a[0][2]) + fabs(a[1][2]);
    if (off == 0.0) break;
    // rolled p/q loops (see k_eigmin6: full unrolling is miscompiled for 6x6)
#pragma unroll 1
    for (int p = 0; p < 2; ++p)
#pragma unroll 1
      for (int q = p + 1; q < 3; ++q) {
        if (a[p][q] == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        const double tt = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(tt * tt + 1.0), sn = tt * c;
        for (int r = 0; r < 3; ++r) {
          const double arp = a[r][p], arq = a[r][q];
          a[r][p] = c * arp - sn * arq;
          a[r][q] = sn * arp + c * arq;
        }
        for (int r = 0; r < 3; ++r) {
          const double apr = a[p][r], aqr = a[q][r];
          a[p][r] = c * apr - sn * aqr;
          a[q][r] = sn * apr + c * aqr;
        }
        a[p][q] = a[q][p] = 0.0;
        for (int r = 0; r < 3; ++r) {
          const double vrp = v[r][p], vrq = v[r][q];
          v[r][p] = c * vrp - sn * vrq;
          v[r][q] = sn * vrp + c * vrq;
        }
      }
  }
  int idx[3] = {0, 1, 2};
  for (int i = 1; i < 3; ++i)
    for (int j = i; j > 0 && a[idx[j]][idx[j]] < a[idx[j - 1]][idx[j - 1]]; --j) {
      const int tmp = idx[j];
      idx[j] = idx[j - 1];
      idx[j - 1] = tmp;
    }
  for (int c = 0; c < 3; ++c) {
    ev[c] = a[idx[c]][idx[c]];
    for (int r = 0; r < 3; ++r) V[3 * c + r] = v[r][idx[c]];
  }
}

struct MatchCfg {
  double gate, huber, plane_tol, plane_ratio, edge_ratio, edge_tol, edge_extent, trim_ratio,
      trim_floor, ground_voxel, ground_radius;
};

__device__ __forceinline__ void line_res(const double p[3], const double q[3], const double d[3],
                                         double r[3]) {
  double J[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) J[3 * i + j] = (i == j ? 1.0 : 0.0) - d[i] * d[j];
  const double e[3] = {p[0] - q[0], p[1] - q[1], p[2] - q[2]};
  for (int i = 0; i < 3; ++i) r[i] = (J[3 * i] * e[0] + J[3 * i + 1] * e[1]) + J[3 * i + 2] * e[2];
}
__device__ __forceinline__ double norm3(const double v[3]) {
  return sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
}

// ground thinning keys: (floor(x/v), floor(y/v)) of ground points passing the
// radius test, first in scan order wins (scan_matcher.cpp:56-68)
__global__ void k_ground_cells(const double* __restrict__ px, const double* __restrict__ py,
                               const double* __restrict__ pz, const uint8_t* __restrict__ kind,
                               size_t n, Pose P, MatchCfg cfg, uint8_t* __restrict__ radius_ok,
                               uint64_t* __restrict__ keys, uint32_t* __restrict__ idx) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  idx[i] = static_cast<uint32_t>(i);
  uint64_t key = ~0ull;
  uint8_t ok = 1;
  if (kind[i] == 2) {
    double x, y, z;
    xform(P, px[i], py[i], pz[i], x, y, z);
    const double dx = x - P.t[0], dy = y - P.t[1];
    if (cfg.ground_radius > 0.0 && sqrt(dx * dx + dy * dy) > cfg.ground_radius) ok = 0;
    if (ok && cfg.ground_voxel > 0.0) {
      const int64_t cx = static_cast<int64_t>(floor(x / cfg.ground_voxel));
      const int64_t cy = static_cast<int64_t>(floor(y / cfg.ground_voxel));
      // the (cx, cy) pair as one key below the ~0 sentinel: cx offset into 31
      // bits, cy into 32 (|cell| < 2^30, far beyond any map extent)
      key = (((static_cast<uint64_t>(cx) + (1ull << 30)) & 0x7fffffffull) << 32) |
            ((static_cast<uint64_t>(cy) + (1ull << 31)) & 0xffffffffull);
    }
  }
  radius_ok[i] = ok;
  keys[i] = key;
}

#ifndef TLG_QG
#define TLG_QG 8
#endif
constexpr int kQG = TLG_QG;  // lanes per query in k_correspond

__global__ void k_correspond(const double* __restrict__ px, const double* __restrict__ py,
                             const double* __restrict__ pz, const uint8_t* __restrict__ kind,
                             size_t n, Pose P, MatchCfg cfg, GridView3 ge, GridView3 gp,
                             const int* __restrict__ lab_e, const int* __restrict__ lab_p,
                             size_t ne, size_t np, const uint8_t* __restrict__ radius_ok,
                             const uint8_t* __restrict__ gfirst, int use_gfirst,
                             const uint32_t* __restrict__ order,
                             uint8_t* __restrict__ pass, int* __restrict__ okind,
                             double* __restrict__ par, double* __restrict__ weight,
                             int* __restrict__ label, double* __restrict__ dist,
                             double* __restrict__ fitq) {
  // one query per group of kQG lanes (knn_group); the fit runs on the
  // group's first lane. Every exit before the search is group-uniform.
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t jj = t / kQG;
  const int glane = static_cast<int>(t % kQG);
  const unsigned gmask = ((1u << kQG) - 1u) << (threadIdx.x & 31 & ~(kQG - 1));
  if (jj >= n) return;
  const size_t i = order[jj];
  if (glane == 0) pass[i] = 0;
  const uint8_t kd = kind[i];
  if (kd == 2 && (!radius_ok[i] || (use_gfirst && !gfirst[i]))) return;
  double pw[3];
  xform(P, px[i], py[i], pz[i], pw[0], pw[1], pw[2]);
  const bool edge = kd == 0;
  const GridView3& g = edge ? ge : gp;
  const int* lab = edge ? lab_e : lab_p;
  if ((edge ? ne : np) == 0) return;
  const double gate2 = cfg.gate * cfg.gate;
  uint32_t ids[8];
  double d2s[8];
  int m;
  if (edge) {
    uint32_t i5[5];
    double d5[5];
    m = knn_group<5, kQG>(g, pw[0], pw[1], pw[2], gate2, glane, gmask, i5, d5);
    if (m < 5 || glane != 0) return;
    for (int a = 0; a < 5; ++a) ids[a] = i5[a];
  } else {
    m = knn_group<8, kQG>(g, pw[0], pw[1], pw[2], gate2, glane, gmask, ids, d2s);
    if (m < 8 || glane != 0) return;
  }
  double cen[3] = {0.0, 0.0, 0.0};
  for (int a = 0; a < m; ++a)
    for (int d = 0; d < 3; ++d) cen[d] += g.pts[3 * ids[a] + d];
  for (int d = 0; d < 3; ++d) cen[d] /= static_cast<double>(m);
  double S[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int a = 0; a < m; ++a) {
    double dv[3];
    for (int d = 0; d < 3; ++d) dv[d] = g.pts[3 * ids[a] + d] - cen[d];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) S[3 * r + c] += dv[r] * dv[c];
  }
  double ev[3], V[9];
  eigen_sym3(S, ev, V);
  // majority label (scan_matcher.cpp:21-33): most frequent, smallest on ties
  int best = -1, best_n = 0;
  for (int a = 0; a < m; ++a) {
    const int l = lab[ids[a]];
    int cnt = 0;
    for (int b = 0; b < m; ++b) cnt += lab[ids[b]] == l;
    if (cnt > best_n || (cnt == best_n && l < best)) {
      best = l;
      best_n = cnt;
    }
  }
  double w = 1.0, dd;
  double* pr = par + 7 * i;
  if (edge) {
    if (ev[2] < cfg.edge_ratio * fmax(ev[1], 1e-12)) return;
    if (ev[2] < cfg.edge_extent * cfg.edge_extent) return;
    double dir[3] = {V[6], V[7], V[8]};
    const double nn = norm3(dir);
    for (int d = 0; d < 3; ++d) dir[d] = dir[d] / nn;
    for (int a = 0; a < m; ++a) {
      double r[3];
      line_res(g.pts + 3 * ids[a], cen, dir, r);
      if (norm3(r) > cfg.edge_tol) return;
    }
    double r[3];
    line_res(pw, cen, dir, r);
    dd = norm3(r);
    if (dd > cfg.gate) return;
    pr[0] = cen[0]; pr[1] = cen[1]; pr[2] = cen[2];
    pr[3] = dir[0]; pr[4] = dir[1]; pr[5] = dir[2]; pr[6] = 0.0;
    fitq[i] = 0.0;
    okind[i] = 0;
  } else {
    if (ev[1] < cfg.plane_ratio * ev[0] || ev[1] < 1e-3) return;
    if (ev[2] > 50.0 * ev[1]) return;
    double nv[3] = {V[0], V[1], V[2]};
    const double nn = norm3(nv);
    for (int d = 0; d < 3; ++d) nv[d] = nv[d] / nn;
    const double off = -((nv[0] * cen[0] + nv[1] * cen[1]) + nv[2] * cen[2]);
    for (int a = 0; a < m; ++a) {
      const double* q = g.pts + 3 * ids[a];
      if (fabs(((nv[0] * q[0] + nv[1] * q[1]) + nv[2] * q[2]) + off) > cfg.plane_tol) return;
    }
    dd = fabs(((nv[0] * pw[0] + nv[1] * pw[1]) + nv[2] * pw[2]) + off);
    if (dd > cfg.gate) return;
    pr[0] = nv[0]; pr[1] = nv[1]; pr[2] = nv[2]; pr[3] = off;
    pr[4] = pr[5] = pr[6] = 0.0;
    fitq[i] = ev[0];
    okind[i] = 1;
  }
  if (cfg.huber > 0.0 && dd > cfg.huber) w = cfg.huber / dd;
  weight[i] = w;
  label[i] = best;
  dist[i] = dd;
  pass[i] = 1;
}

__global__ void k_query_keys(const double* __restrict__ px, const double* __restrict__ py,
                             const double* __restrict__ pz, const uint8_t* __restrict__ kind,
                             size_t n, Pose P, GridView3 ge, GridView3 gp, int cell_bits,
                             uint64_t* __restrict__ keys, uint32_t* __restrict__ idx) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double q[3];
  xform(P, px[i], py[i], pz[i], q[0], q[1], q[2]);
  const bool edge = kind[i] == 0;
  const GridView3& g = edge ? ge : gp;
  uint64_t cell = 0;
  if (g.dim[0] > 0) {
    int c[3];
    for (int a = 0; a < 3; ++a)
      c[a] = min(max(static_cast<int>(floor((q[a] - g.org[a]) / g.cell)), 0), g.dim[a] - 1);
    cell = static_cast<uint64_t>((c[2] * g.dim[1] + c[1]) * g.dim[0] + c[0]);
  }
  keys[i] = (static_cast<uint64_t>(edge ? 0 : 1) << cell_bits) | cell;
  idx[i] = static_cast<uint32_t>(i);
}

// order-preserving signed double -> unsigned key (radix sort of fitq)
__device__ __forceinline__ uint64_t dkey(double v) {
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
  return (b >> 63) ? ~b : (b | (1ull << 63));
}

__global__ void k_sel_keys(const uint32_t* __restrict__ sel, size_t cnt,
                           const double* __restrict__ dist, const double* __restrict__ fitq,
                           const int* __restrict__ kind, uint64_t* __restrict__ kd,
                           uint64_t* __restrict__ kq, int* __restrict__ nplane) {
  const size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (j >= cnt) return;
  const uint32_t i = sel[j];
  kd[j] = dkey(dist[i]);
  const bool plane = kind[i] == 1;
  kq[j] = plane ? dkey(fitq[i]) : ~0ull;  // edges sort after every plane
  if (plane) atomicAdd(nplane, 1);
}

__device__ __forceinline__ double undkey(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & ~(1ull << 63)) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

// scan_matcher.cpp:150-180 trims with the order statistics read on the
// device (sorted keys kd2 / kq2, plane count): no host round trip
__global__ void k_trim(const uint32_t* __restrict__ sel, size_t cnt, const double* __restrict__ dist,
                       const double* __restrict__ fitq, const uint64_t* __restrict__ kd2,
                       const uint64_t* __restrict__ kq2, const int* __restrict__ nplane,
                       double trim_ratio, double trim_floor, uint8_t* __restrict__ keep) {
  const size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (j >= cnt) return;
  const double cut = fmax(__dmul_rn(trim_ratio, undkey(kd2[cnt / 2])), trim_floor);
  const int np = *nplane;
  const double qcut = np > 0 ? fmax(__dmul_rn(10.0, undkey(kq2[np / 2])), 1e-7) : INFINITY;
  const uint32_t i = sel[j];
  keep[j] = dist[i] <= cut && fitq[i] <= qcut;
}

__global__ void k_pack_corr(const uint32_t* __restrict__ sel, size_t cnt,
                            const double* __restrict__ px, const double* __restrict__ py,
                            const double* __restrict__ pz, const int* __restrict__ kind,
                            const double* __restrict__ par, const double* __restrict__ weight,
                            const int* __restrict__ label, const double* __restrict__ dist,
                            const double* __restrict__ fitq, int* __restrict__ ck,
                            uint32_t* __restrict__ cf, double* __restrict__ cp,
                            double* __restrict__ cw, int* __restrict__ cl,
                            double* __restrict__ cd, double* __restrict__ cq,
                            double* __restrict__ cps) {
  const size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (j >= cnt) return;
  const uint32_t i = sel[j];
  ck[j] = kind[i];
  cf[j] = i;
  for (int a = 0; a < 7; ++a) cp[7 * j + a] = par[7 * i + a];
  cw[j] = weight[i];
  cl[j] = label[i];
  cd[j] = dist[i];
  cq[j] = fitq[i];
  cps[3 * j] = px[i];
  cps[3 * j + 1] = py[i];
  cps[3 * j + 2] = pz[i];
}

// total_cost feature rows (scan_matcher.cpp:196-214) -> 29 sums per block,
// fixed-order tree; rows as in the oracle
constexpr int kNeThreads = 128;
__global__ void __launch_bounds__(kNeThreads) k_feature_ne(size_t nc, const int* __restrict__ ck,
                                                           const double* __restrict__ ps,
                                                           const double* __restrict__ par,
                                                           const double* __restrict__ wgt, Pose P,
                                                           double* __restrict__ partials) {
  __shared__ double red[29][kNeThreads];
  double acc[29];
  for (int e = 0; e < 29; ++e) acc[e] = 0.0;
  for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < nc;
       j += (size_t)gridDim.x * blockDim.x) {
    const double s0 = ps[3 * j], s1 = ps[3 * j + 1], s2 = ps[3 * j + 2];
    double pw[3];
    xform(P, s0, s1, s2, pw[0], pw[1], pw[2]);
    const double H[9] = {0.0, -s2, s1, s2, 0.0, -s0, -s1, s0, 0.0};
    double dp[3][6];
    for (int i = 0; i < 3; ++i)
      for (int c = 0; c < 3; ++c) {
        dp[i][c] = (-P.R[3 * i] * H[c] + -P.R[3 * i + 1] * H[3 + c]) + -P.R[3 * i + 2] * H[6 + c];
        dp[i][3 + c] = (i == c) ? 1.0 : 0.0;
      }
    const double sw = sqrt(wgt[j]);
    const double* pr = par + 7 * j;
    auto add_row = [&](double r, const double (&Jr)[6]) {
      int k = 0;
      for (int a = 0; a < 6; ++a)
        for (int b = a; b < 6; ++b) acc[k++] += Jr[a] * Jr[b];
      for (int a = 0; a < 6; ++a) acc[21 + a] += Jr[a] * r;
      acc[27] += r * r;
      acc[28] += 1.0;
    };
    if (ck[j] == 0) {
      const double d[3] = {pr[3], pr[4], pr[5]};
      double J[9];
      for (int i = 0; i < 3; ++i)
        for (int c = 0; c < 3; ++c) J[3 * i + c] = (i == c ? 1.0 : 0.0) - d[i] * d[c];
      const double e[3] = {pw[0] - pr[0], pw[1] - pr[1], pw[2] - pr[2]};
      for (int i = 0; i < 3; ++i) {
        const double rv = (J[3 * i] * e[0] + J[3 * i + 1] * e[1]) + J[3 * i + 2] * e[2];
        double Jr[6];
        for (int c = 0; c < 6; ++c)
          Jr[c] = sw * ((J[3 * i] * dp[0][c] + J[3 * i + 1] * dp[1][c]) + J[3 * i + 2] * dp[2][c]);
        add_row(sw * rv, Jr);
      }
    } else {
      const double rv = ((pr[0] * pw[0] + pr[1] * pw[1]) + pr[2] * pw[2]) + pr[3];
      double Jr[6];
      for (int c = 0; c < 6; ++c)
        Jr[c] = sw * ((pr[0] * dp[0][c] + pr[1] * dp[1][c]) + pr[2] * dp[2][c]);
      add_row(sw * rv, Jr);
    }
  }
  for (int e = 0; e < 29; ++e) red[e][threadIdx.x] = acc[e];
  __syncthreads();
  if (threadIdx.x < 29) {
    double v = 0.0;
    for (int t = 0; t < kNeThreads; ++t) v += red[threadIdx.x][t];
    partials[blockIdx.x * 29 + threadIdx.x] = v;
  }
}

// total_cost feature rows materialised (scan_matcher.cpp:196-214): the rows
// of correspondence j start at row0[j] (3 for an edge, 1 for a plane); J is
// column-major rows x 6 (Eigen's CostEval layout, ld = rows). Same
// arithmetic as k_feature_ne, which reduces these rows.
__global__ void k_feature_rows(size_t nc, const int* __restrict__ ck, const double* __restrict__ ps,
                               const double* __restrict__ par, const double* __restrict__ wgt,
                               const uint32_t* __restrict__ row0, Pose P, size_t rows,
                               double* __restrict__ r_out, double* __restrict__ J_out) {
  const size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (j >= nc) return;
  const double s0 = ps[3 * j], s1 = ps[3 * j + 1], s2 = ps[3 * j + 2];
  double pw[3];
  xform(P, s0, s1, s2, pw[0], pw[1], pw[2]);
  const double H[9] = {0.0, -s2, s1, s2, 0.0, -s0, -s1, s0, 0.0};
  double dp[3][6];
  for (int i = 0; i < 3; ++i)
    for (int c = 0; c < 3; ++c) {
      dp[i][c] = (-P.R[3 * i] * H[c] + -P.R[3 * i + 1] * H[3 + c]) + -P.R[3 * i + 2] * H[6 + c];
      dp[i][3 + c] = (i == c) ? 1.0 : 0.0;
    }
  const double sw = sqrt(wgt[j]);
  const double* pr = par + 7 * j;
  const size_t o = row0[j];
  if (ck[j] == 0) {
    const double d[3] = {pr[3], pr[4], pr[5]};
    double J[9];
    for (int i = 0; i < 3; ++i)
      for (int c = 0; c < 3; ++c) J[3 * i + c] = (i == c ? 1.0 : 0.0) - d[i] * d[c];
    const double e[3] = {pw[0] - pr[0], pw[1] - pr[1], pw[2] - pr[2]};
    for (int i = 0; i < 3; ++i) {
      r_out[o + i] = sw * ((J[3 * i] * e[0] + J[3 * i + 1] * e[1]) + J[3 * i + 2] * e[2]);
      for (int c = 0; c < 6; ++c)
        J_out[o + i + c * rows] =
            sw * ((J[3 * i] * dp[0][c] + J[3 * i + 1] * dp[1][c]) + J[3 * i + 2] * dp[2][c]);
    }
  } else {
    r_out[o] = sw * (((pr[0] * pw[0] + pr[1] * pw[1]) + pr[2] * pw[2]) + pr[3]);
    for (int c = 0; c < 6; ++c)
      J_out[o + c * rows] = sw * ((pr[0] * dp[0][c] + pr[1] * dp[1][c]) + pr[2] * dp[2][c]);
  }
}

template <typename T>
size_t select_flagged(tlg_ctx* ctx, const uint8_t* flags, size_t n, uint32_t* out) {
  cudaStream_t s = ctx->stream;
  int* d_cnt = ctx->ws<int>(S_COUNT, 1);
  thrust::counting_iterator<uint32_t> it(0);
  size_t tmp = 0;
  TLG_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, it, flags, out, d_cnt, n, s));
  void* d = ctx->ws<char>(S_CUB2, tmp);
  TLG_CUDA(cub::DeviceSelect::Flagged(d, tmp, it, flags, out, d_cnt, n, s));
  int h = 0;
  TLG_CUDA(cudaMemcpyAsync(&h, d_cnt, sizeof(int), cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
  return static_cast<size_t>(h);
}

// first element per key run (stable sort keeps scan order inside a run)
void first_per_key(tlg_ctx* ctx, uint64_t* keys, uint32_t* idx, size_t n, uint8_t* first,
                   bool sentinel) {
  cudaStream_t s = ctx->stream;
  uint64_t* keys2 = ctx->ws<uint64_t>(S_KEYS2, n);
  uint32_t* idx2 = ctx->ws<uint32_t>(S_VALS2, n);
  size_t tmp = 0;
  TLG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, keys2, idx, idx2, n, 0, 64, s));
  void* d = ctx->ws<char>(S_CUB, tmp);
  TLG_CUDA(cub::DeviceRadixSort::SortPairs(d, tmp, keys, keys2, idx, idx2, n, 0, 64, s));
  TLG_CUDA(cudaMemsetAsync(first, 0, n, s));
  k_first_of_run<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(keys2, idx2, n, sentinel ? 1 : 0,
                                                             first);
  TLG_LAUNCHED(ctx);
}

__global__ void k_bbox(const double* __restrict__ pts, size_t n, double* __restrict__ out) {
  __shared__ double sh[6][1024];
  double v[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
  for (size_t i = threadIdx.x; i < n; i += blockDim.x)
    for (int a = 0; a < 3; ++a) {
      v[a] = fmin(v[a], pts[3 * i + a]);
      v[3 + a] = fmax(v[3 + a], pts[3 * i + a]);
    }
  for (int a = 0; a < 6; ++a) sh[a][threadIdx.x] = v[a];
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o)
      for (int a = 0; a < 6; ++a)
        sh[a][threadIdx.x] = a < 3 ? fmin(sh[a][threadIdx.x], sh[a][threadIdx.x + o])
                                   : fmax(sh[a][threadIdx.x], sh[a][threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x < 6) out[threadIdx.x] = sh[threadIdx.x][0];
}

__global__ void k_compose(const uint32_t* __restrict__ sel, const uint32_t* __restrict__ sel2,
                          size_t c2, uint32_t* __restrict__ out) {
  const size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (j < c2) out[j] = sel[sel2[j]];
}

__global__ void k_sum29(const double* __restrict__ partials, int blocks, double* __restrict__ out) {
  const int k = threadIdx.x;
  if (k >= 29) return;
  double v = 0.0;
  for (int b = 0; b < blocks; ++b) v += partials[b * 29 + k];
  out[k] = v;
}

void build_grid(tlg_map* m, int cls, double gate) {
  tlg_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  auto& G = m->grid[cls];
  const size_t n = m->n[cls];
  if (G.gate == gate) return;
  G.gate = gate;
  if (n == 0) {
    G.dim[0] = G.dim[1] = G.dim[2] = 0;
    return;
  }
  // bounding box (device reduction; the host only sizes the grid from it)
  double* bb = ctx->ws<double>(S_PARTIALS, 6);
  k_bbox<<<1, 1024, 0, s>>>(m->pts[cls].p, n, bb);
  TLG_LAUNCHED(ctx);
  double hb[6];
  TLG_CUDA(cudaMemcpyAsync(hb, bb, sizeof(hb), cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
  const double lo[3] = {hb[0], hb[1], hb[2]}, hi[3] = {hb[3], hb[4], hb[5]};
  // cell edge for ~12 points per occupied cell (shell search, knn_grid), not
  // above the gate, at most 256 cells per axis
  double ext = 0.0, vol = 1.0;
  for (int a = 0; a < 3; ++a) {
    ext = std::max(ext, hi[a] - lo[a]);
    vol *= std::max(hi[a] - lo[a], 1e-3);
  }
  // ~12 points per cell for a volumetric cloud, or for a surface cloud
  // (LiDAR maps are mostly surfaces: area ~ the bounding box's face sum)
  const double e0 = std::max(hi[0] - lo[0], 1e-3), e1 = std::max(hi[1] - lo[1], 1e-3),
               e2 = std::max(hi[2] - lo[2], 1e-3);
  const double c3 = std::cbrt(vol * 12.0 / static_cast<double>(n));
  const double c2 = std::sqrt((e0 * e1 + e0 * e2 + e1 * e2) * 12.0 / static_cast<double>(n));
  G.cell = std::max(std::min(std::min(c3, c2), gate), ext / 256.0);
  if (!(G.cell > 0.0)) G.cell = 1.0;
  for (int a = 0; a < 3; ++a) {
    G.org[a] = lo[a];
    G.dim[a] = static_cast<int>(std::floor((hi[a] - lo[a]) / G.cell)) + 1;
  }
  const size_t cells = static_cast<size_t>(G.dim[0]) * G.dim[1] * G.dim[2];
  uint32_t* keys = ctx->ws<uint32_t>(S_TKEYS, n);
  uint32_t* keys2 = ctx->ws<uint32_t>(S_NODE_IDX, n);
  uint32_t* idx = ctx->ws<uint32_t>(S_VALS, n);
  G.ids.ensure(n);
  GridView3 gv{m->pts[cls].p, nullptr, nullptr, {G.org[0], G.org[1], G.org[2]}, G.cell,
               {G.dim[0], G.dim[1], G.dim[2]}};
  k_cell_keys<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(m->pts[cls].p, n, gv, keys, idx);
  TLG_LAUNCHED(ctx);
  size_t tmp = 0;
  TLG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, keys2, idx, G.ids.p, n, 0, 32, s));
  void* d = ctx->ws<char>(S_CUB, tmp);
  TLG_CUDA(cub::DeviceRadixSort::SortPairs(d, tmp, keys, keys2, idx, G.ids.p, n, 0, 32, s));
  G.start.ensure(cells + 1);
  int* cnt = ctx->ws<int>(S_ROWOF, cells + 1);
  TLG_CUDA(cudaMemsetAsync(cnt, 0, (cells + 1) * sizeof(int), s));
  k_cell_count<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(keys, n, cnt);
  TLG_LAUNCHED(ctx);
  size_t tmp2 = 0;
  TLG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp2, cnt, G.start.p, cells + 1, s));
  void* d2 = ctx->ws<char>(S_CUB2, tmp2);
  TLG_CUDA(cub::DeviceScan::ExclusiveSum(d2, tmp2, cnt, G.start.p, cells + 1, s));
}

GridView3 grid_view3(tlg_map* m, int cls) {
  auto& G = m->grid[cls];
  return GridView3{m->pts[cls].p, G.start.p, G.ids.p, {G.org[0], G.org[1], G.org[2]}, G.cell,
                   {G.dim[0], G.dim[1], G.dim[2]}};
}

}  // namespace

tlg_map* map_new(tlg_ctx* ctx, double voxel, size_t window) {
  auto* m = new tlg_map;
  m->ctx = ctx;
  m->voxel = voxel;
  m->window = window;
  return m;
}

void map_free(tlg_map* m) {
  if (!m) return;
  cudaStreamSynchronize(m->ctx->stream);
  delete m;
}

tlg_ctx* map_ctx(tlg_map* m) { return m->ctx; }

size_t map_points_host(tlg_map* m, int kind, double* xyz, int32_t* labels, size_t cap) {
  const size_t n = m->n[kind], k = std::min(n, cap);
  if (k && xyz)
    TLG_CUDA(cudaMemcpyAsync(xyz, m->pts[kind].p, 3 * k * 8, cudaMemcpyDeviceToHost, m->ctx->stream));
  if (k && labels)
    TLG_CUDA(cudaMemcpyAsync(labels, m->lab[kind].p, k * 4, cudaMemcpyDeviceToHost, m->ctx->stream));
  TLG_CUDA(cudaStreamSynchronize(m->ctx->stream));
  return n;
}

size_t correspondences_host(tlg_map* m, int32_t* kind, uint32_t* feature, double* params,
                            double* weight, int32_t* label, double* dist, double* fitq,
                            size_t cap) {
  cudaStream_t s = m->ctx->stream;
  const size_t k = std::min(m->nc, cap);
  if (k) {
    if (kind) TLG_CUDA(cudaMemcpyAsync(kind, m->c_kind.p, k * 4, cudaMemcpyDeviceToHost, s));
    if (feature) TLG_CUDA(cudaMemcpyAsync(feature, m->c_feat.p, k * 4, cudaMemcpyDeviceToHost, s));
    if (params) TLG_CUDA(cudaMemcpyAsync(params, m->c_par.p, 7 * k * 8, cudaMemcpyDeviceToHost, s));
    if (weight) TLG_CUDA(cudaMemcpyAsync(weight, m->c_w.p, k * 8, cudaMemcpyDeviceToHost, s));
    if (label) TLG_CUDA(cudaMemcpyAsync(label, m->c_lab.p, k * 4, cudaMemcpyDeviceToHost, s));
    if (dist) TLG_CUDA(cudaMemcpyAsync(dist, m->c_dist.p, k * 8, cudaMemcpyDeviceToHost, s));
    if (fitq) TLG_CUDA(cudaMemcpyAsync(fitq, m->c_q.p, k * 8, cudaMemcpyDeviceToHost, s));
  }
  TLG_CUDA(cudaStreamSynchronize(s));
  return m->nc;
}

void map_insert(tlg_map* m, const double* px, const double* py, const double* pz,
                const uint8_t* kind, const int* label, size_t n, const double R[9],
                const double t[3]) {
  tlg_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  Pose P;
  for (int i = 0; i < 9; ++i) P.R[i] = R[i];
  for (int i = 0; i < 3; ++i) P.t[i] = t[i];
  tlg_map::Frame fr;
  if (n) {
    double* xyz = ctx->ws<double>(S_WORK1, 3 * n);
    uint64_t* keys = ctx->ws<uint64_t>(S_KEYS, n);
    uint32_t* idx = ctx->ws<uint32_t>(S_VALS, n);
    uint8_t* first = ctx->ws<uint8_t>(S_NODE_FLAG, n);
    uint8_t* flag = ctx->ws<uint8_t>(S_BLOCKFLAG, n);
    uint32_t* sel = ctx->ws<uint32_t>(S_MERGED, n);
    k_map_keys<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(px, py, pz, kind, n, P, m->voxel, xyz,
                                                          keys, idx);
    TLG_LAUNCHED(ctx);
    first_per_key(ctx, keys, idx, n, first, false);  // every (kind, voxel) key is valid
    for (int cls = 0; cls < 2; ++cls) {
      k_flag_class<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(first, kind, n, cls, flag);
      TLG_LAUNCHED(ctx);
      const size_t cnt = select_flagged<uint32_t>(ctx, flag, n, sel);
      fr.n[cls] = cnt;
      fr.pts[cls].ensure(3 * std::max<size_t>(cnt, 1));
      fr.lab[cls].ensure(std::max<size_t>(cnt, 1));
      if (cnt) {
        k_gather_pts<<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(sel, cnt, xyz, label,
                                                                   fr.pts[cls].p, fr.lab[cls].p);
        TLG_LAUNCHED(ctx);
      }
    }
  }
  m->frames.push_back(std::move(fr));
  while (m->frames.size() > m->window) m->frames.pop_front();
  // rebuild (local_map.cpp:47-60): concatenate the window, frame order
  for (int cls = 0; cls < 2; ++cls) {
    size_t tot = 0;
    for (const auto& f : m->frames) tot += f.n[cls];
    m->pts[cls].ensure(3 * std::max<size_t>(tot, 1));
    m->lab[cls].ensure(std::max<size_t>(tot, 1));
    size_t off = 0;
    for (const auto& f : m->frames) {
      if (f.n[cls]) {
        TLG_CUDA(cudaMemcpyAsync(m->pts[cls].p + 3 * off, f.pts[cls].p, 3 * f.n[cls] * 8,
                                 cudaMemcpyDeviceToDevice, s));
        TLG_CUDA(cudaMemcpyAsync(m->lab[cls].p + off, f.lab[cls].p, f.n[cls] * 4,
                                 cudaMemcpyDeviceToDevice, s));
      }
      off += f.n[cls];
    }
    m->n[cls] = tot;
    m->grid[cls].gate = -1.0;  // rebuilt lazily for the query gate
  }
  TLG_CUDA(cudaStreamSynchronize(s));
}

size_t build_correspondences_device(tlg_map* m, const double* px, const double* py,
                                    const double* pz, const uint8_t* kind, size_t n,
                                    const double R[9], const double t[3], const double cfgv[11]) {
  tlg_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  m->nc = 0;
  if (n == 0 || m->n[0] + m->n[1] == 0) return 0;
  Pose P;
  for (int i = 0; i < 9; ++i) P.R[i] = R[i];
  for (int i = 0; i < 3; ++i) P.t[i] = t[i];
  const MatchCfg cfg{cfgv[0], cfgv[1], cfgv[2], cfgv[3], cfgv[4],  cfgv[5],
                     cfgv[6], cfgv[7], cfgv[8], cfgv[9], cfgv[10]};
  build_grid(m, 0, cfg.gate);
  build_grid(m, 1, cfg.gate);
  const unsigned nb = static_cast<unsigned>((n + 127) / 128);
  // ground thinning
  uint8_t* rok = ctx->ws<uint8_t>(S_ACTIVE, n);
  uint8_t* gfirst = ctx->ws<uint8_t>(S_NODE_FLAG, n);
  uint64_t* keys = ctx->ws<uint64_t>(S_KEYS, n);
  uint32_t* idx = ctx->ws<uint32_t>(S_VALS, n);
  k_ground_cells<<<nb, 128, 0, s>>>(px, py, pz, kind, n, P, cfg, rok, keys, idx);
  TLG_LAUNCHED(ctx);
  const int use_gfirst = cfg.ground_voxel > 0.0;
  if (use_gfirst) first_per_key(ctx, keys, idx, n, gfirst, true);
  // per-feature fits
  uint8_t* pass = ctx->ws<uint8_t>(S_BLOCKFLAG, n);
  int* okind = ctx->ws<int>(S_ROWPTR, n);
  double* par = ctx->ws<double>(S_WORK2, 7 * n);
  double* wgt = ctx->ws<double>(S_OUT_R, n);
  int* lab = ctx->ws<int>(S_COLIDX, n);
  double* dist = ctx->ws<double>(S_OUT_GX, n);
  double* fq = ctx->ws<double>(S_OUT_GY, n);
  // process features in (kind, map cell) order: neighbouring threads share
  // cells and loop trip counts (results are still indexed by feature)
  uint64_t* qk = ctx->ws<uint64_t>(S_KEYS, n);
  uint32_t* qi = ctx->ws<uint32_t>(S_VALS, n);
  uint64_t* qk2 = ctx->ws<uint64_t>(S_KEYS2, n);
  uint32_t* order = ctx->ws<uint32_t>(S_VALS2, n);
  // key = kind bit above the cell index: sort only the bits in use
  int cell_bits = 1;
  for (int cls = 0; cls < 2; ++cls) {
    const GridView3 gv = grid_view3(m, cls);
    const uint64_t nc = static_cast<uint64_t>(std::max(gv.dim[0], 0)) * std::max(gv.dim[1], 0) *
                        std::max(gv.dim[2], 0);
    while (cell_bits < 62 && (1ull << cell_bits) < nc) ++cell_bits;
  }
  k_query_keys<<<nb, 128, 0, s>>>(px, py, pz, kind, n, P, grid_view3(m, 0), grid_view3(m, 1),
                                  cell_bits, qk, qi);
  TLG_LAUNCHED(ctx);
  size_t tmpq = 0;
  TLG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmpq, qk, qk2, qi, order, n, 0, cell_bits + 1,
                                           s));
  void* dq = ctx->ws<char>(S_CUB, tmpq);
  TLG_CUDA(cub::DeviceRadixSort::SortPairs(dq, tmpq, qk, qk2, qi, order, n, 0, cell_bits + 1, s));
  k_correspond<<<static_cast<unsigned>((n * kQG + 127) / 128), 128, 0, s>>>(
      px, py, pz, kind, n, P, cfg, grid_view3(m, 0), grid_view3(m, 1),
                                  m->lab[0].p, m->lab[1].p, m->n[0], m->n[1], rok, gfirst,
                                  use_gfirst, order, pass, okind, par, wgt, lab, dist, fq);
  TLG_LAUNCHED(ctx);
  uint32_t* sel = ctx->ws<uint32_t>(S_MERGED, n);
  size_t cnt = select_flagged<uint32_t>(ctx, pass, n, sel);
  if (cnt == 0) return 0;
  // adaptive trims (scan_matcher.cpp:150-180): exact order statistics
  if (cfg.trim_ratio > 0.0) {
    uint64_t* kd = ctx->ws<uint64_t>(S_KEYS, cnt);
    uint64_t* kq = ctx->ws<uint64_t>(S_KEYS2, cnt);
    uint64_t* kd2 = ctx->ws<uint64_t>(S_TROWP, cnt);
    uint64_t* kq2 = ctx->ws<uint64_t>(S_SOLVE, cnt);
    int* nplane = ctx->ws<int>(S_FLAGS, 4);
    TLG_CUDA(cudaMemsetAsync(nplane, 0, sizeof(int), s));
    k_sel_keys<<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(sel, cnt, dist, fq, okind, kd, kq,
                                                             nplane);
    TLG_LAUNCHED(ctx);
    size_t tmp = 0;
    TLG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, kd, kd2, cnt, 0, 64, s));
    void* d = ctx->ws<char>(S_CUB, tmp);
    TLG_CUDA(cub::DeviceRadixSort::SortKeys(d, tmp, kd, kd2, cnt, 0, 64, s));
    TLG_CUDA(cub::DeviceRadixSort::SortKeys(d, tmp, kq, kq2, cnt, 0, 64, s));
    uint8_t* keep = ctx->ws<uint8_t>(S_ACTIVE, cnt);
    k_trim<<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(sel, cnt, dist, fq, kd2, kq2, nplane,
                                                         cfg.trim_ratio, cfg.trim_floor, keep);
    TLG_LAUNCHED(ctx);
    uint32_t* sel2 = ctx->ws<uint32_t>(S_NODE_IDX, cnt);
    const size_t c2 = select_flagged<uint32_t>(ctx, keep, cnt, sel2);
    uint32_t* sel3 = ctx->ws<uint32_t>(S_TKEYS, std::max<size_t>(c2, 1));
    if (c2) {
      k_compose<<<(unsigned)((c2 + 255) / 256), 256, 0, s>>>(sel, sel2, c2, sel3);
      TLG_LAUNCHED(ctx);
    }
    sel = sel3;
    cnt = c2;
  }
  m->c_kind.ensure(std::max<size_t>(cnt, 1));
  m->c_feat.ensure(std::max<size_t>(cnt, 1));
  m->c_par.ensure(7 * std::max<size_t>(cnt, 1));
  m->c_w.ensure(std::max<size_t>(cnt, 1));
  m->c_lab.ensure(std::max<size_t>(cnt, 1));
  m->c_dist.ensure(std::max<size_t>(cnt, 1));
  m->c_q.ensure(std::max<size_t>(cnt, 1));
  m->c_ps.ensure(3 * std::max<size_t>(cnt, 1));
  if (cnt) {
    k_pack_corr<<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(
        sel, cnt, px, py, pz, okind, par, wgt, lab, dist, fq, m->c_kind.p, m->c_feat.p,
        m->c_par.p, m->c_w.p, m->c_lab.p, m->c_dist.p, m->c_q.p, m->c_ps.p);
    TLG_LAUNCHED(ctx);
  }
  TLG_CUDA(cudaStreamSynchronize(s));
  m->nc = cnt;
  return cnt;
}

void feature_rows_device(tlg_ctx* ctx, size_t nc, const int32_t* kind, const double* ps,
                         const double* par, const double* wgt, const double R[9], const double t[3],
                         double* r, double* J, size_t* rows_out) {
  cudaStream_t s = ctx->stream;
  std::vector<uint32_t> row0(nc);
  size_t rows = 0;
  for (size_t j = 0; j < nc; ++j) {
    row0[j] = static_cast<uint32_t>(rows);
    rows += kind[j] == 0 ? 3 : 1;
  }
  *rows_out = rows;
  if (nc == 0) return;
  int* dk = ctx->ws<int>(S_KEYS, nc);
  double* dps = ctx->ws<double>(S_NODES_X, 3 * nc);
  double* dpar = ctx->ws<double>(S_NODES_Y, 7 * nc);
  double* dw = ctx->ws<double>(S_VALS, nc);
  uint32_t* dr0 = ctx->ws<uint32_t>(S_VALS2, nc);
  double* dr = ctx->ws<double>(S_OUT_R, rows);
  double* dJ = ctx->ws<double>(S_OUT_J, 6 * rows);
  TLG_CUDA(cudaMemcpyAsync(dk, kind, nc * 4, cudaMemcpyHostToDevice, s));
  TLG_CUDA(cudaMemcpyAsync(dps, ps, 3 * nc * 8, cudaMemcpyHostToDevice, s));
  TLG_CUDA(cudaMemcpyAsync(dpar, par, 7 * nc * 8, cudaMemcpyHostToDevice, s));
  TLG_CUDA(cudaMemcpyAsync(dw, wgt, nc * 8, cudaMemcpyHostToDevice, s));
  TLG_CUDA(cudaMemcpyAsync(dr0, row0.data(), nc * 4, cudaMemcpyHostToDevice, s));
  Pose P;
  for (int i = 0; i < 9; ++i) P.R[i] = R[i];
  for (int i = 0; i < 3; ++i) P.t[i] = t[i];
  k_feature_rows<<<(unsigned)((nc + 127) / 128), 128, 0, s>>>(nc, dk, dps, dpar, dw, dr0, P, rows, dr,
                                                              dJ);
  TLG_LAUNCHED(ctx);
  TLG_CUDA(cudaMemcpyAsync(r, dr, rows * 8, cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaMemcpyAsync(J, dJ, 6 * rows * 8, cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
}

void feature_normal_eq_device(tlg_map* m, const double R[9], const double t[3], double ne29[29]) {
  tlg_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  for (int k = 0; k < 29; ++k) ne29[k] = 0.0;
  if (m->nc == 0) return;
  Pose P;
  for (int i = 0; i < 9; ++i) P.R[i] = R[i];
  for (int i = 0; i < 3; ++i) P.t[i] = t[i];
  const int blocks = static_cast<int>(std::min<size_t>((m->nc + kNeThreads - 1) / kNeThreads, static_cast<size_t>(ctx->num_sms)));
  double* partials = ctx->ws<double>(S_PARTIALS, static_cast<size_t>(blocks) * 29);
  k_feature_ne<<<blocks, kNeThreads, 0, s>>>(m->nc, m->c_kind.p, m->c_ps.p, m->c_par.p, m->c_w.p,
                                             P, partials);
  TLG_LAUNCHED(ctx);
  double* out = ctx->ws<double>(S_SOLVE, 29);
  k_sum29<<<1, 32, 0, s>>>(partials, blocks, out);
  TLG_LAUNCHED(ctx);
  TLG_CUDA(cudaMemcpyAsync(ne29, out, 29 * 8, cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
}

namespace {
// scan_matcher.cpp:300-305: delta = -(A + mu diag(A)^+ + 1e-3 I)^-1 g with a
// diagonally pivoted LDL^T (Eigen::LDLT's algorithm, as restated in the
// oracle). One thread: 6 x 6.
__global__ void k_lm_step(const double* __restrict__ ne29, double mu, double* __restrict__ out) {
  double a[6][6];
  int k = 0;
  for (int i = 0; i < 6; ++i)
    for (int j = i; j < 6; ++j) {
      a[i][j] = ne29[k];
      a[j][i] = ne29[k];
      ++k;
    }
  for (int i = 0; i < 6; ++i) a[i][i] += mu * fmax(a[i][i], 1e-12);
  for (int i = 0; i < 6; ++i) a[i][i] += 1e-3;
  int perm[6];
  double tmp[6];
  for (int kk = 0; kk < 6; ++kk) {
    int big = kk;
    double bv = fabs(a[kk][kk]);
    for (int i = kk + 1; i < 6; ++i)
      if (fabs(a[i][i]) > bv) {
        bv = fabs(a[i][i]);
        big = i;
      }
    perm[kk] = big;
    if (big != kk) {
      for (int c = 0; c < kk; ++c) { const double t = a[kk][c]; a[kk][c] = a[big][c]; a[big][c] = t; }
      for (int r = big + 1; r < 6; ++r) { const double t = a[r][kk]; a[r][kk] = a[r][big]; a[r][big] = t; }
      { const double t = a[kk][kk]; a[kk][kk] = a[big][big]; a[big][big] = t; }
      for (int i = kk + 1; i < big; ++i) { const double t = a[i][kk]; a[i][kk] = a[big][i]; a[big][i] = t; }
    }
    if (kk > 0) {
      for (int c = 0; c < kk; ++c) tmp[c] = a[c][c] * a[kk][c];
      double sacc = 0.0;
      for (int c = 0; c < kk; ++c) sacc += a[kk][c] * tmp[c];
      a[kk][kk] -= sacc;
      for (int r = kk + 1; r < 6; ++r) {
        double acc = 0.0;
        for (int c = 0; c < kk; ++c) acc += a[r][c] * tmp[c];
        a[r][kk] -= acc;
      }
    }
    const double akk = a[kk][kk];
    if (kk == 0 && !(fabs(akk) > 0.0)) {
      for (int j = 0; j < 6; ++j) perm[j] = j;
      break;
    }
    if (kk + 1 < 6 && fabs(akk) > 0.0)
      for (int r = kk + 1; r < 6; ++r) a[r][kk] /= akk;
  }
  double v[6];
  for (int i = 0; i < 6; ++i) v[i] = ne29[21 + i];
  for (int kk = 0; kk < 6; ++kk) { const double t = v[kk]; v[kk] = v[perm[kk]]; v[perm[kk]] = t; }
  for (int kk = 0; kk < 6; ++kk)
    for (int r = kk + 1; r < 6; ++r) v[r] -= a[r][kk] * v[kk];
  for (int kk = 0; kk < 6; ++kk) {
    const double d = a[kk][kk];
    v[kk] = (fabs(d) > 2.2250738585072014e-308) ? v[kk] / d : 0.0;
  }
  for (int kk = 5; kk >= 0; --kk) {
    double sacc = v[kk];
    for (int r = kk + 1; r < 6; ++r) sacc -= a[r][kk] * v[r];
    v[kk] = sacc;
  }
  for (int kk = 5; kk >= 0; --kk) { const double t = v[kk]; v[kk] = v[perm[kk]]; v[perm[kk]] = t; }
  bool finite = true;
  for (int i = 0; i < 6; ++i) {
    out[i] = -v[i];
    finite = finite && isfinite(out[i]);
  }
  out[6] = finite ? 1.0 : 0.0;
}
}  // namespace

bool lm_step_device(tlg_ctx* ctx, const double ne29[29], double mu, double delta[6]) {
  cudaStream_t s = ctx->stream;
  double* d = ctx->ws<double>(S_SOLVE, 40);
  TLG_CUDA(cudaMemcpyAsync(d, ne29, 29 * 8, cudaMemcpyHostToDevice, s));
  k_lm_step<<<1, 1, 0, s>>>(d, mu, d + 32);
  TLG_LAUNCHED(ctx);
  double h[7];
  TLG_CUDA(cudaMemcpyAsync(h, d + 32, 7 * 8, cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < 6; ++i) delta[i] = h[i];
  return h[6] != 0.0;
}

namespace {
// smallest eigenvalue of the symmetric 6x6 J^T J (cyclic Jacobi); the
// degeneracy probe of lm_solve (scan_matcher.cpp:280-287)
__global__ void k_eigmin6(const double* __restrict__ ne29, double* __restrict__ out) {
  double a[6][6];
  int k = 0;
  for (int i = 0; i < 6; ++i)
    for (int j = i; j < 6; ++j) {
      a[i][j] = ne29[k];
      a[j][i] = ne29[k];
      ++k;
    }
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < 6; ++p)
      for (int q = p + 1; q < 6; ++q) off += fabs(a[p][q]);
    if (off == 0.0) break;
    // rolled p/q loops: nvcc 12.9's full unrolling of this in-place rotation
    // miscompiles (wrong eigenvalues; correct with -Xcicc -O0) — keep rolled
#pragma unroll 1
    for (int p = 0; p < 5; ++p)
#pragma unroll 1
      for (int q = p + 1; q < 6; ++q) {
        if (a[p][q] == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        const double tt = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(tt * tt + 1.0), sn = tt * c;
        for (int r = 0; r < 6; ++r) {
          const double arp = a[r][p], arq = a[r][q];
          a[r][p] = c * arp - sn * arq;
          a[r][q] = sn * arp + c * arq;
        }
        for (int r = 0; r < 6; ++r) {
          const double apr = a[p][r], aqr = a[q][r];
          a[p][r] = c * apr - sn * aqr;
          a[q][r] = sn * apr + c * aqr;
        }
        a[p][q] = a[q][p] = 0.0;
      }
  }
  double mn = a[0][0];
  for (int i = 1; i < 6; ++i) mn = fmin(mn, a[i][i]);
  out[0] = mn;
}
}  // namespace

double eigmin6_device(tlg_ctx* ctx, const double ne29[29]) {
  cudaStream_t s = ctx->stream;
  double* d = ctx->ws<double>(S_SOLVE, 40);
  TLG_CUDA(cudaMemcpyAsync(d, ne29, 29 * 8, cudaMemcpyHostToDevice, s));
  k_eigmin6<<<1, 1, 0, s>>>(d, d + 32);
  TLG_LAUNCHED(ctx);
  double h = 0.0;
  TLG_CUDA(cudaMemcpyAsync(&h, d + 32, 8, cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
  return h;
}

}  // namespace tlg
