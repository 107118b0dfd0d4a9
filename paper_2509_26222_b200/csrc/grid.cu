// K1 centre_hash_build: GridIndex2 (grid_index.hpp:16-66) over the model's
// centres as a dense CSR cell array in HBM. Cell coordinates use the
// reference's exact expression static_cast<int>(floor(v / cell)); ids stay
// ascending inside each cell (stable radix sort), and centre coordinates
// and weights are stored in cell order so a 3x3 cell sweep reads contiguous
// runs.
#include <cub/cub.cuh>

#include <climits>
#include <cmath>

#include "internal.cuh"

namespace tlg {

__global__ void k_cell_coords(const double* __restrict__ cx, const double* __restrict__ cy,
                              size_t n, double cell, int* __restrict__ ix, int* __restrict__ iy,
                              int* __restrict__ bbox) {
  int mnx = INT_MAX, mny = INT_MAX, mxx = INT_MIN, mxy = INT_MIN;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const int a = static_cast<int>(floor(cx[i] / cell));
    const int b = static_cast<int>(floor(cy[i] / cell));
    ix[i] = a;
    iy[i] = b;
    mnx = min(mnx, a);
    mny = min(mny, b);
    mxx = max(mxx, a);
    mxy = max(mxy, b);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mnx = min(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
    mny = min(mny, __shfl_xor_sync(0xffffffffu, mny, o));
    mxx = max(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
    mxy = max(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&bbox[0], mnx);
    atomicMin(&bbox[1], mny);
    atomicMax(&bbox[2], mxx);
    atomicMax(&bbox[3], mxy);
  }
}

__global__ void k_cell_linear(const int* __restrict__ ix, const int* __restrict__ iy, size_t n,
                              int gx0, int gy0, int gny, uint32_t* __restrict__ key,
                              uint32_t* __restrict__ id, int* __restrict__ counts) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t k = static_cast<uint32_t>(ix[i] - gx0) * static_cast<uint32_t>(gny) +
                     static_cast<uint32_t>(iy[i] - gy0);
  key[i] = k;
  id[i] = static_cast<uint32_t>(i);
  atomicAdd(&counts[k], 1);
}

__global__ void k_gather_sorted(const uint32_t* __restrict__ sid, size_t n,
                                const double* __restrict__ cx, const double* __restrict__ cy,
                                const double* __restrict__ w, double* __restrict__ scx,
                                double* __restrict__ scy, double* __restrict__ sw) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t j = sid[i];
  if (scx) scx[i] = cx[j];
  if (scy) scy[i] = cy[j];
  sw[i] = w[j];
}

// ---------------------------------------------------------------------------
// Lattice detection: centre (cx, cy) is node (i, j) iff it equals
// min + i * res bit-exactly (center_select.cpp:55-56), i = llround((c-min)/res).
__global__ void k_lattice_check(const double* __restrict__ cx, const double* __restrict__ cy,
                                size_t n, double min_x, double min_y, double res,
                                int* __restrict__ st) {
  for (size_t c = blockIdx.x * (size_t)blockDim.x + threadIdx.x; c < n;
       c += (size_t)gridDim.x * blockDim.x) {
    const double fi = (cx[c] - min_x) / res, fj = (cy[c] - min_y) / res;
    bool ok = fabs(fi) < 1e8 && fabs(fj) < 1e8;
    int i = 0, j = 0;
    if (ok) {
      i = static_cast<int>(llround(fi));
      j = static_cast<int>(llround(fj));
      ok = __dadd_rn(min_x, __dmul_rn(static_cast<double>(i), res)) == cx[c] &&
           __dadd_rn(min_y, __dmul_rn(static_cast<double>(j), res)) == cy[c];
    }
    if (!ok) {
      atomicOr(&st[0], 1);
    } else {
      atomicMin(&st[1], i);
      atomicMin(&st[2], j);
      atomicMax(&st[3], i);
      atomicMax(&st[4], j);
    }
  }
}

__global__ void k_lattice_fill(const double* __restrict__ cx, const double* __restrict__ cy,
                               const double* __restrict__ w, size_t n, double min_x,
                               double min_y, double res, int i_org, int j_org, int nj,
                               double* __restrict__ W, double* __restrict__ W1,
                               int* __restrict__ P, int* __restrict__ slot,
                               int* __restrict__ dup) {
  for (size_t c = blockIdx.x * (size_t)blockDim.x + threadIdx.x; c < n;
       c += (size_t)gridDim.x * blockDim.x) {
    const int i = static_cast<int>(llround((cx[c] - min_x) / res)) - i_org;
    const int j = static_cast<int>(llround((cy[c] - min_y) / res)) - j_org;
    const int s = i * nj + j;
    slot[c] = s;
    W[s] = w[c];
    W1[s + 1] = w[c];
    if (atomicAdd(&P[s], 1) != 0) atomicOr(dup, 1);
  }
}

__global__ void k_lattice_axes(double min_v, double res, int org, int count, double cell,
                               AxisNode* __restrict__ ax) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  const double v = __dadd_rn(min_v, __dmul_rn(static_cast<double>(k + org), res));
  ax[k] = AxisNode{v, static_cast<int>(floor(v / cell)), 0};
}

__global__ void k_lattice_ranges(const AxisNode* __restrict__ ax, int count, int span, int qbase,
                                 int nq, int2* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nq) return;
  auto first = [&](long long c) {  // first node with cell >= c
    int lo = 0, hi = count;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (ax[mid].cell < c) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  const long long q = static_cast<long long>(qbase) + t;
  out[t] = make_int2(first(q - span), first(q + span + 1));
}

// Range table over every point cell whose sweep can reach a node, plus a
// margin; cells outside clamp to an end entry, whose range is empty.
static void lattice_ranges(tlg_model* m, const DBuf<AxisNode>& ax, int count, double mn, int org,
                           DBuf<int2>& out, int& base, int& nq) {
  const double res = m->cparams.mesh_resolution, cell = m->grid.cell;
  const int span = m->grid.span;
  const double v0 = mn + static_cast<double>(org) * res;
  const double v1 = mn + static_cast<double>(org + count - 1) * res;
  const long long c0 = static_cast<long long>(std::floor(v0 / cell)) - span - 3;
  const long long c1 = static_cast<long long>(std::floor(v1 / cell)) + span + 3;
  require(c1 - c0 < (1ll << 24) && c0 > INT_MIN / 2 && c1 < INT_MAX / 2, TLG_RUNTIME_ERROR,
          "lattice cell range too large");
  base = static_cast<int>(c0);
  nq = static_cast<int>(c1 - c0 + 1);
  out.ensure(nq);
  k_lattice_ranges<<<(nq + 127) / 128, 128, 0, m->ctx->stream>>>(ax.p, count, span, base, nq,
                                                                  out.p);
  TLG_LAUNCHED(m->ctx);
}

// Per-cell LOOSE flags (eval.cu): bit 0 = the cell's four corner nodes are
// present (every point of the cell is supported); bit 1 = for every point of
// the cell the boundary pairs summed without the cutoff test move z by at
// most 1e-10 of the parity scale sum |w kappa| and a gradient component by at
// most 1e-10 of sum |w kappa| d / sigma^2. The worst case of the skipped
// tests is n_bd kappa(cutoff) |w|max (times cutoff / sigma^2 for the
// gradient, since d kappa(d) falls beyond sigma). The scales are bounded
// below on each of kSub x kSub sub-cells by the window's inside pairs: |w|
// times the minimum over the sub-cell of kappa (and of kappa d) for that pair
// offset (pairlb, host-computed per geometry); the cell's bound is the
// smallest sub-cell bound.
constexpr int kSub = 4;
__global__ void k_cell_flags(const double* __restrict__ W, const int* __restrict__ P, int ni, int nj,
                             int lo, int win, const double* __restrict__ pairlb, double loose_k,
                             double loose_d, uint8_t* __restrict__ out) {
  const size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (e >= (size_t)ni * nj) return;
  const int i = static_cast<int>(e / nj), j = static_cast<int>(e % nj);
  const int i0 = i - lo, j0 = j - lo;
  uint8_t f = 0;
  if (i0 >= 0 && j0 >= 0 && i0 + win <= ni && j0 + win <= nj) {
    const size_t c = static_cast<size_t>(i) * nj + j;
    if (P[c] && P[c + 1] && P[c + nj] && P[c + nj + 1]) f |= 1;
    double wmax = 0.0;
    double ls[kSub * kSub], lt[kSub * kSub];
    for (int q = 0; q < kSub * kSub; ++q) ls[q] = lt[q] = 0.0;
    const int np = win * win;
    for (int k = 0; k < win; ++k)
      for (int l = 0; l < win; ++l) {
        const double w = fabs(W[static_cast<size_t>(i0 + k) * nj + j0 + l]);
        wmax = fmax(wmax, w);
        const double* lb = pairlb + 2 * (k * win + l);
        for (int q = 0; q < kSub * kSub; ++q) {
          ls[q] = fma(w, lb[2 * q * np], ls[q]);
          lt[q] = fma(w, lb[2 * q * np + 1], lt[q]);
        }
      }
    double ms = ls[0], mt = lt[0];
    for (int q = 1; q < kSub * kSub; ++q) {
      ms = fmin(ms, ls[q]);
      mt = fmin(mt, lt[q]);
    }
    const double err = loose_k * wmax;
    if (err <= 1e-10 * ms && err * loose_d <= 1e-10 * mt) f |= 2;
  }
  out[e] = f;
}

// pairlb for the model's geometry: window pair (k, l) is the node at
// (a, b) = (k - lo, l - lo) cells from the base cell's origin; a point of
// sub-cell (u, v) lies in [u/kSub, (u+1)/kSub) x [...] cells, so its |dx| to
// the node spans the interval of |a - x| over that range.
static void pair_lower_bounds(const tlg_model* m, std::vector<double>& lb) {
  const LatticeGrid& L = m->lat;
  const double res = m->cparams.mesh_resolution, c = m->kc.neg_inv_2s2;
  const int np = L.win * L.win;
  lb.assign(static_cast<size_t>(2 * np * kSub * kSub), 0.0);
  auto span = [](int a, double x0, double x1, double& lo, double& hi) {
    // |a - x| for x in [x0, x1]
    const double d0 = std::fabs(a - x0), d1 = std::fabs(a - x1);
    hi = std::max(d0, d1);
    lo = (a >= x0 && a <= x1) ? 0.0 : std::min(d0, d1);
  };
  for (int u = 0; u < kSub; ++u)
    for (int v = 0; v < kSub; ++v) {
      const int q = u * kSub + v;
      for (int k = 0; k < L.win; ++k)
        for (int l = 0; l < L.win; ++l) {
          if (!((L.inmask[k] >> l) & 1u)) continue;
          double xl, xh, yl, yh;
          span(k - L.lo, double(u) / kSub, double(u + 1) / kSub, xl, xh);
          span(l - L.lo, double(v) / kSub, double(v + 1) / kSub, yl, yh);
          const double dmin = res * std::sqrt(xl * xl + yl * yl);
          const double dmax = res * std::sqrt(xh * xh + yh * yh);
          const double kmin = std::exp(c * dmax * dmax);
          const double kdmin = std::min(std::exp(c * dmin * dmin) * dmin, kmin * dmax);
          double* o = lb.data() + 2 * (q * np + k * L.win + l);
          o[0] = kmin * (1.0 - 1e-12);
          o[1] = kdmin * (1.0 - 1e-12);
        }
    }
}

int prepare_sweep(tlg_model* m) {
  const int kind = sweep_kind(m);
  LatticeGrid& L = m->lat;
  if (kind >= 200 && L.wmax_dirty) {
    const size_t nn = static_cast<size_t>(L.ni) * L.nj;
    L.cflag.ensure(nn);
    std::vector<double> lb;
    pair_lower_bounds(m, lb);
    L.pairlb.ensure(lb.size());
    TLG_CUDA(cudaMemcpyAsync(L.pairlb.p, lb.data(), lb.size() * sizeof(double), cudaMemcpyHostToDevice,
                             m->ctx->stream));
    const LatticeView v = lattice_view(m);
    const unsigned b = static_cast<unsigned>((nn + 255) / 256);
    k_cell_flags<<<b, 256, 0, m->ctx->stream>>>(L.W.p, L.P.p, L.ni, L.nj, L.lo, L.win, L.pairlb.p, v.loose_k,
                                                v.loose_d, L.cflag.p);
    TLG_LAUNCHED(m->ctx);
    // the host vector is read by the async copy: wait before it goes out of scope
    TLG_CUDA(cudaStreamSynchronize(m->ctx->stream));
    L.wmax_dirty = false;
  }
  return kind;
}

__global__ void k_lattice_refresh(const int* __restrict__ slot, const double* __restrict__ w,
                                  size_t n, double* __restrict__ W, double* __restrict__ W1) {
  const size_t c = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (c < n) {
    W[slot[c]] = w[c];
    W1[slot[c] + 1] = w[c];
  }
}

// Window geometry and pair classes (host: ~WIN^2 scalar parameter setup).
static bool lattice_geometry(tlg_model* m, LatticeGrid& L) {
  const double res = m->cparams.mesh_resolution;
  if (!(res > 0.0)) return false;
  const double R = m->kernel.cutoff_radius / res;  // cutoff in lattice units
  if (!(R > 0.0) || R + 2 > kMaxWin) return false;
  const Geom g = make_geom(R);
  if (g.win == 0) return false;
  L.lo = g.lo;
  L.win = g.win;
  L.pad = L.win + 1;
  for (int k = 0; k < 16; ++k) {
    L.inmask[k] = g.in[k];
    L.bdmask[k] = g.bd[k];
  }
  L.geom_id = -1;
  for (int i = 0; i < kNumGeoms; ++i)
    if (geom_equal(g, kGeoms[i])) L.geom_id = i;
  const int c0 = L.lo, c1 = L.lo + 1;
  L.corner_ok = ((L.inmask[c0] >> c0) & 1) && ((L.inmask[c0] >> c1) & 1) &&
                ((L.inmask[c1] >> c0) & 1) && ((L.inmask[c1] >> c1) & 1);
  return true;
}

static void build_lattice(tlg_model* m) {
  tlg_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  LatticeGrid& L = m->lat;
  L.valid = false;
  const size_t n = m->hcx.size();
  if (n == 0 || !lattice_geometry(m, L)) return;
  const double res = m->cparams.mesh_resolution;
  const double mnx = m->cparams.roi_min_x, mny = m->cparams.roi_min_y;
  int* st = ctx->ws<int>(S_COUNT, 8);
  const int hs[8] = {0, INT_MAX, INT_MAX, INT_MIN, INT_MIN, 0, 0, 0};
  TLG_CUDA(cudaMemcpyAsync(st, hs, sizeof(hs), cudaMemcpyHostToDevice, s));
  const unsigned blocks = static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 4ull * ctx->num_sms));
  k_lattice_check<<<blocks, 256, 0, s>>>(m->cx.p, m->cy.p, n, mnx, mny, res, st);
  TLG_LAUNCHED(ctx);
  int h[8];
  TLG_CUDA(cudaMemcpyAsync(h, st, sizeof(h), cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
  if (h[0]) return;
  L.i_org = h[1] - L.pad;
  L.j_org = h[2] - L.pad;
  const long long ni = static_cast<long long>(h[3]) - h[1] + 1 + 2 * L.pad;
  long long nj = static_cast<long long>(h[4]) - h[2] + 1 + 2 * L.pad;
  nj += nj & 1;  // even row pitch: a column's pair alignment is that of its base
  if (ni * nj > (1ll << 28)) return;
  L.ni = static_cast<int>(ni);
  L.nj = static_cast<int>(nj);
  const size_t nn = static_cast<size_t>(ni * nj);
  L.W.ensure(nn + 2);
  L.W1.ensure(nn + 2);
  L.P.ensure(nn);
  L.slot.ensure(n);
  TLG_CUDA(cudaMemsetAsync(L.W.p, 0, (nn + 2) * sizeof(double), s));
  TLG_CUDA(cudaMemsetAsync(L.W1.p, 0, (nn + 2) * sizeof(double), s));
  TLG_CUDA(cudaMemsetAsync(L.P.p, 0, nn * sizeof(int), s));
  int* dup = st + 5;
  k_lattice_fill<<<blocks, 256, 0, s>>>(m->cx.p, m->cy.p, m->w.p, n, mnx, mny, res, L.i_org,
                                        L.j_org, L.nj, L.W.p, L.W1.p, L.P.p, L.slot.p, dup);
  TLG_LAUNCHED(ctx);
  L.ax.ensure(L.ni);
  L.ay.ensure(L.nj);
  const double cell = m->grid.cell;
  k_lattice_axes<<<(L.ni + 127) / 128, 128, 0, s>>>(mnx, res, L.i_org, L.ni, cell, L.ax.p);
  TLG_LAUNCHED(ctx);
  k_lattice_axes<<<(L.nj + 127) / 128, 128, 0, s>>>(mny, res, L.j_org, L.nj, cell, L.ay.p);
  TLG_LAUNCHED(ctx);
  lattice_ranges(m, L.ax, L.ni, mnx, L.i_org, L.xr, L.xr_base, L.xr_n);
  lattice_ranges(m, L.ay, L.nj, mny, L.j_org, L.yr, L.yr_base, L.yr_n);
  L.min_x = mnx;
  L.min_y = mny;
  L.wmax_dirty = true;
  int hd = 0;
  TLG_CUDA(cudaMemcpyAsync(&hd, dup, sizeof(int), cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
  if (hd) return;  // repeated node: keep the generic sweep
  L.org_x = mnx + static_cast<double>(L.i_org) * res;
  L.org_y = mny + static_cast<double>(L.j_org) * res;
  L.inv_res = 1.0 / res;
  L.valid = true;
}

LatticeView lattice_view(const tlg_model* m) {
  const LatticeGrid& L = m->lat;
  LatticeView v;
  v.W = L.W.p;
  v.W1 = L.W1.p;
  v.P = L.P.p;
  v.ax = L.ax.p;
  v.ay = L.ay.p;
  v.xr = L.xr.p;
  v.yr = L.yr.p;
  v.xr_base = L.xr_base;
  v.xr_n = L.xr_n;
  v.yr_base = L.yr_base;
  v.yr_n = L.yr_n;
  v.i_org = L.i_org;
  v.j_org = L.j_org;
  v.min_x = L.min_x;
  v.min_y = L.min_y;
  v.ni = L.ni;
  v.nj = L.nj;
  v.lo = L.lo;
  v.span = m->grid.span;
  v.org_x = L.org_x;
  v.org_y = L.org_y;
  v.inv_res = L.inv_res;
  v.cell = m->grid.cell;
  for (int k = 0; k < 16; ++k) {
    v.inmask[k] = L.inmask[k];
    v.bdmask[k] = L.bdmask[k];
  }
  v.corner_ok = L.corner_ok;
  // e_y recurrence (eval.cu): exponents stay within +-600 over the window
  // span, so no under/overflow; otherwise evaluate exp per node.
  const double res = m->cparams.mesh_resolution;
  const double c = m->kc.neg_inv_2s2;
  const double span = (L.win + 1) * res;
  v.res = res;
  v.c_res = c * res;
  v.k2 = std::exp(2.0 * c * res * res);
  v.rec_ok = (std::fabs(c) * span * span < 600.0 && std::fabs(c) * res * 2.0 * span < 600.0) ? 1 : 0;
  // LOOSE path (eval.cu): n_bd boundary pairs, each failing one lies at
  // d > cutoff and adds at most kcut |w| to z and, since d kappa(d) falls for
  // d > sigma, kcut cutoff |w| / sigma^2 to a gradient component. Enabled
  // when kappa at the cutoff is small enough that the per-point check passes
  // for ordinary (smooth) weights.
  int nbd = 0;
  for (int k = 0; k < 16; ++k) nbd += __builtin_popcount(L.bdmask[k]);
  const double kcut = std::exp(m->kc.r2 * c);
  const double sigma = m->kernel.sigma, rho = m->kernel.cutoff_radius;
  v.loose_k = nbd * kcut;
  v.loose_d = rho;
  v.loose_ok = (rho > sigma && v.loose_k * std::max(1.0, rho / sigma) <= 1e-11) ? 1 : 0;
  v.cflag = L.cflag.p;
  return v;
}

void build_center_grid(tlg_model* m) {
  tlg_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  CenterGrid& g = m->grid;
  const size_t n = m->hcx.size();
  g.cell = std::min(m->kernel.cutoff_radius, 1e6);  // terrain_model.cpp:63
  g.span = static_cast<int>(std::ceil(m->kernel.cutoff_radius / g.cell));
  if (n == 0) {
    g.gx0 = g.gy0 = 0;
    g.gnx = g.gny = 0;
    g.cell_start.ensure(2);
    TLG_CUDA(cudaMemsetAsync(g.cell_start.p, 0, 2 * sizeof(int), s));
    m->grid_dirty = false;
    return;
  }
  int* ix = ctx->ws<int>(S_KEYS, n);
  int* iy = ctx->ws<int>(S_KEYS2, n);
  int* bbox = ctx->ws<int>(S_COUNT, 4);
  const int hb[4] = {INT_MAX, INT_MAX, INT_MIN, INT_MIN};
  TLG_CUDA(cudaMemcpyAsync(bbox, hb, sizeof(hb), cudaMemcpyHostToDevice, s));
  const unsigned blocks = static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 4ull * ctx->num_sms));
  k_cell_coords<<<blocks, 256, 0, s>>>(m->cx.p, m->cy.p, n, g.cell, ix, iy, bbox);
  TLG_LAUNCHED(ctx);
  int hbox[4];
  TLG_CUDA(cudaMemcpyAsync(hbox, bbox, sizeof(hbox), cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
  g.gx0 = hbox[0];
  g.gy0 = hbox[1];
  const long long gnx = static_cast<long long>(hbox[2]) - hbox[0] + 1;
  const long long gny = static_cast<long long>(hbox[3]) - hbox[1] + 1;
  require(gnx * gny <= (1ll << 27), TLG_RUNTIME_ERROR,
          "centre spread too large for the dense centre grid");
  g.gnx = static_cast<int>(gnx);
  g.gny = static_cast<int>(gny);
  const size_t ncell = static_cast<size_t>(gnx * gny);

  g.cell_start.ensure(ncell + 1);
  TLG_CUDA(cudaMemsetAsync(g.cell_start.p, 0, (ncell + 1) * sizeof(int), s));
  uint32_t* key = ctx->ws<uint32_t>(S_VALS, n);
  uint32_t* key2 = ctx->ws<uint32_t>(S_VALS2, n);
  uint32_t* id = ctx->ws<uint32_t>(S_NODE_IDX, n);
  g.sorted_id.ensure(n);
  k_cell_linear<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ix, iy, n, g.gx0, g.gy0, g.gny, key,
                                                           id, g.cell_start.p);
  TLG_LAUNCHED(ctx);
  // stable radix sort by cell -> ids ascending within a cell
  int end_bit = 1;
  while (end_bit < 32 && (1ull << end_bit) < ncell) ++end_bit;
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, key2, id, g.sorted_id.p, (int)n, 0, end_bit, s);
  void* dtmp = ctx->ws<unsigned char>(S_CUB, tmp);
  TLG_CUDA(cub::DeviceRadixSort::SortPairs(dtmp, tmp, key, key2, id, g.sorted_id.p, (int)n, 0,
                                           end_bit, s));
  ++ctx->launches;
  // counts -> exclusive starts (in place over ncell+1 entries)
  tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, g.cell_start.p, g.cell_start.p, (int)(ncell + 1), s);
  dtmp = ctx->ws<unsigned char>(S_CUB, tmp);
  TLG_CUDA(cub::DeviceScan::ExclusiveSum(dtmp, tmp, g.cell_start.p, g.cell_start.p,
                                         (int)(ncell + 1), s));
  ++ctx->launches;
  g.scx.ensure(n);
  g.scy.ensure(n);
  g.sw.ensure(n);
  k_gather_sorted<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g.sorted_id.p, n, m->cx.p, m->cy.p,
                                                             m->w.p, g.scx.p, g.scy.p, g.sw.p);
  TLG_LAUNCHED(ctx);
  build_lattice(m);
  m->grid_dirty = false;
}

void ensure_grid(tlg_model* m) {
  if (m->grid_dirty) build_center_grid(m);
}

void sync_weights_to_grid(tlg_model* m) {
  if (m->grid_dirty) {
    build_center_grid(m);
    return;
  }
  const size_t n = m->hcx.size();
  if (n == 0) return;
  k_gather_sorted<<<(unsigned)((n + 255) / 256), 256, 0, m->ctx->stream>>>(
      m->grid.sorted_id.p, n, m->cx.p, m->cy.p, m->w.p, nullptr, nullptr, m->grid.sw.p);
  TLG_LAUNCHED(m->ctx);
  if (m->lat.valid) {
    k_lattice_refresh<<<(unsigned)((n + 255) / 256), 256, 0, m->ctx->stream>>>(m->lat.slot.p, m->w.p,
                                                                          n, m->lat.W.p,
                                                                          m->lat.W1.p);
    TLG_LAUNCHED(m->ctx);
    m->lat.wmax_dirty = true;
  }
}

GridView grid_view(const tlg_model* m) {
  const CenterGrid& g = m->grid;
  return GridView{g.scx.p, g.scy.p, g.sw.p, g.sorted_id.p, g.cell_start.p, g.cell,
                  g.span,  g.gx0,   g.gy0,  g.gnx,         g.gny};
}

}  // namespace tlg
