// Lattice element assembly of the batch-ridge system (terrain_model.cpp:
// 269-308: H = lambda I + Mt Mt^T, b = Mt z) on the FP64 tensor pipe.
//
// When the centres are mesh nodes (the select_centers / birth case, the
// LatticeGrid of grid.cu), every observation in lattice cell (ib, jb) has its
// features among the same WIN x WIN node window. The observations are sorted
// by cell (stable radix sort: a deterministic order), and per cell the dense
// feature block F (points x [WIN^2 nodes | z]) is built in shared memory —
// exactly the reference's membership: the per-pair no-FMA d^2 <= r^2 test,
// the hash-cell window of GridIndex2::radius_query (the xr / yr ranges of the
// lattice), absent nodes zero. The cell's Gram F^T F, whose z row is the
// cell's part of b, runs as 8x8 DMMA tiles (m8n8k4, lower triangle only):
// each point costs WIN^4 / 2 tensor FMAs instead of the row-wise Gram's
// shared-memory read-modify-writes, and each observation is read once instead
// of once per feature.
//
// Cells are walked in columns: a CTA owns lattice column ib and a segment of
// its cells (ascending jb) and adds each cell's Gram into its own slice of a
// node-major scratch Hlat[colour][node][offset] (offset = the partner's
// (di, dj), di <= 0, lower in lattice order). colour = (ib mod WIN, segment
// parity): CTAs of one colour touch disjoint node windows, so no atomics, and
// a final pass sums the colours in a fixed order into the band storage of H
// (merged rows, update.cu BatchPlan). Every step has a fixed order, so the
// result is bit-reproducible run to run (tests/test_gpu_stress.py).
#include <cub/cub.cuh>
#include <math_constants.h>

#include <cstdlib>

#include "internal.cuh"

namespace tlg {

namespace {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int WIN>
struct LatGeo {
  static constexpr int kF = WIN * WIN;                          // node features per cell
  static constexpr int kNT = (kF + 1 + 7) / 8;                  // 8-wide tiles (+ the z column)
  static constexpr int kNW = (kNT + 1) / 2;                     // DMMA warps: tile rows w and kNT-1-w
  static constexpr int kWarps = kNW > 8 ? kNW : 8;              // CTA warps (all build features)
  static constexpr int kFP = ((kNT * 8 - 4 + 15) / 16) * 16 + 4;  // F pitch = 4 (mod 16): no bank conflicts
  static constexpr int kKO = WIN * (2 * WIN - 1);               // partner offsets per node
  static constexpr int kPPW = 32 / WIN;                         // points per warp and batch
  static constexpr int kBatch = kWarps * kPPW;                  // points per F block
  static constexpr int kRows = (kBatch + 3) / 4 * 4;            // F rows (whole k-steps)
  static constexpr size_t kSmem = sizeof(double) * (2 * kRows * kFP + 2 * kWarps * kPPW * WIN) +
                                  sizeof(uint32_t) * WIN;
};

// Cell key of each observation, the eval's window base (eval.cu
// eval_lattice: ib = floor((x - org) / res)); observations whose window
// leaves the padded lattice have no centre within the cutoff (sorted last).
__global__ void k_lat_keys(LatticeView L, int win, const double* __restrict__ x,
                           const double* __restrict__ y, size_t n, uint32_t skip,
                           uint32_t* __restrict__ key, uint32_t* __restrict__ idx) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t k = skip;
  const double fx = floor((x[i] - L.org_x) * L.inv_res), fy = floor((y[i] - L.org_y) * L.inv_res);
  if (fx >= L.lo && fy >= L.lo && fx - L.lo + win <= L.ni && fy - L.lo + win <= L.nj)
    k = static_cast<uint32_t>(fx) * static_cast<uint32_t>(L.nj) + static_cast<uint32_t>(fy);
  key[i] = k;
  idx[i] = static_cast<uint32_t>(i);
}

// start[c] = first sorted observation with key >= c, c in [0, cells]
__global__ void k_lat_bounds(const uint32_t* __restrict__ key, size_t n, uint32_t cells,
                             uint32_t* __restrict__ start) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > cells) return;
  size_t lo = 0, hi = n;
  while (lo < hi) {
    const size_t mid = (lo + hi) >> 1;
    if (key[mid] < c) lo = mid + 1; else hi = mid;
  }
  start[c] = static_cast<uint32_t>(lo);
}

// Observations in cell order, with each one's reference cell-window masks
// (GridIndex2::radius_query's (2 span + 1)^2 cells, the xr / yr ranges of the
// lattice): bit k (x) / 16 + k (y) set when window node i0 + k / j0 + k lies
// in a candidate cell — computed once here (a division per axis) instead of
// per node in the assembly.
__global__ void k_lat_gather(LatticeView L, int win, const uint32_t* __restrict__ perm,
                             const uint32_t* __restrict__ key, uint32_t skip, size_t n,
                             const double* __restrict__ x, const double* __restrict__ y,
                             const double* __restrict__ z, double* __restrict__ ox,
                             double* __restrict__ oy, double* __restrict__ oz,
                             uint32_t* __restrict__ om) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t j = perm[i];
  const double px = x[j], py = y[j];
  ox[i] = px;
  oy[i] = py;
  oz[i] = z[j];
  uint32_t m = 0;
  const uint32_t k = key[i];
  if (k != skip) {
    const int i0 = static_cast<int>(k / static_cast<uint32_t>(L.nj)) - L.lo;
    const int j0 = static_cast<int>(k % static_cast<uint32_t>(L.nj)) - L.lo;
    const int qx = static_cast<int>(floor(px / L.cell)), qy = static_cast<int>(floor(py / L.cell));
    const int2 rx = L.xr[min(max(qx - L.xr_base, 0), L.xr_n - 1)];
    const int2 ry = L.yr[min(max(qy - L.yr_base, 0), L.yr_n - 1)];
    for (int a = 0; a < win; ++a) {
      if (i0 + a >= rx.x && i0 + a < rx.y) m |= 1u << a;
      if (j0 + a >= ry.x && j0 + a < ry.y) m |= 1u << (16 + a);
    }
  }
  om[i] = m;
}

// Warp W's DMMA over one F block: tile rows R1 = W and R2 = kNT-1-W, lower
// tiles only (acc[t] = (R1, t), acc[R1+1+t] = (R2, t)); all indices are
// compile-time, so the accumulators stay in registers.
template <int WIN, int W>
__device__ __forceinline__ void lat_mma(const double* __restrict__ F, int ksteps, double (&acc)[LatGeo<WIN>::kNT + 1][2]) {
  using G = LatGeo<WIN>;
  constexpr int R1 = W, R2 = G::kNT - 1 - W;
  const int lane = threadIdx.x & 31;
  const double* f = F + (lane & 3) * G::kFP + (lane >> 2);
  for (int ks = 0; ks < ksteps; ++ks, f += 4 * G::kFP) {
    double fr[R2 + 1];
#pragma unroll
    for (int t = 0; t <= R2; ++t) fr[t] = f[8 * t];
#pragma unroll
    for (int t = 0; t <= R1; ++t) dmma884(acc[t][0], acc[t][1], fr[R1], fr[t]);
    if constexpr (R2 != R1) {
#pragma unroll
      for (int t = 0; t <= R2; ++t) dmma884(acc[R1 + 1 + t][0], acc[R1 + 1 + t][1], fr[R2], fr[t]);
    }
  }
}

// Address in the colour slice of the cell's Gram entry (u, v), u >= v in
// window order: node pairs at Hc[lower node][offset], the z row at
// bc[node]; nullptr for upper / padding entries.
template <int WIN>
__device__ __forceinline__ double* lat_slot(int u, int v, int i0, int j0, int nj,
                                            double* __restrict__ Hc, double* __restrict__ bc) {
  using G = LatGeo<WIN>;
  if (u < v || v >= G::kF) return nullptr;
  if (u >= G::kF)
    return u == G::kF ? bc + (i0 + v / WIN) * static_cast<size_t>(nj) + j0 + v % WIN : nullptr;
  const int iu = u / WIN, ju = u % WIN, iv = v / WIN, jv = v % WIN;
  const size_t a = (i0 + iu) * static_cast<size_t>(nj) + (j0 + ju);
  return Hc + a * G::kKO + (iv - iu + WIN - 1) * (2 * WIN - 1) + (jv - ju + WIN - 1);
}

// Adds the warp's accumulators to the colour slice. Every (u, v) of a cell
// is a distinct entry, so the read-modify-writes of a group of tiles are
// issued as independent loads first (one L2 round trip per group, not per
// entry); groups and cells stay ordered by program order and the barriers.
template <int WIN, int W>
__device__ __forceinline__ void lat_flush(double (&acc)[LatGeo<WIN>::kNT + 1][2], int i0, int j0,
                                          int nj, double* __restrict__ Hc, double* __restrict__ bc) {
  using G = LatGeo<WIN>;
  constexpr int R1 = W, R2 = G::kNT - 1 - W;
  constexpr int kTiles = R2 != R1 ? G::kNT + 1 : R1 + 1;
  constexpr int kGroup = 4;  // tiles per group: 8 loads in flight per lane
  const int lane = threadIdx.x & 31;
  const int m = lane >> 2, n0 = 2 * (lane & 3);
#pragma unroll
  for (int g0 = 0; g0 < kTiles; g0 += kGroup) {
    double* p[2 * kGroup];
    double v[2 * kGroup];
#pragma unroll
    for (int q = 0; q < kGroup; ++q) {
      const int s = g0 + q;
      if (s < kTiles) {
        const int row = s <= R1 ? R1 : R2, col = s <= R1 ? s : s - R1 - 1;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          p[2 * q + e] = acc[s][e] != 0.0 ? lat_slot<WIN>(8 * row + m, 8 * col + n0 + e, i0, j0, nj, Hc, bc)
                                          : nullptr;
        }
      } else {
        p[2 * q] = p[2 * q + 1] = nullptr;
      }
    }
#pragma unroll
    for (int q = 0; q < 2 * kGroup; ++q) v[q] = p[q] ? *p[q] : 0.0;
#pragma unroll
    for (int q = 0; q < 2 * kGroup; ++q)
      if (p[q]) *p[q] = v[q] + acc[g0 + q / 2 < kTiles ? g0 + q / 2 : 0][q & 1];
  }
}

template <int WIN, int W = 0>
__device__ __forceinline__ void lat_mma_any(int w, const double* F, int ksteps,
                                            double (&acc)[LatGeo<WIN>::kNT + 1][2]) {
  if constexpr (W < LatGeo<WIN>::kNW) {
    if (w == W) lat_mma<WIN, W>(F, ksteps, acc);
    else lat_mma_any<WIN, W + 1>(w, F, ksteps, acc);
  }
}

template <int WIN, int W = 0>
__device__ __forceinline__ void lat_flush_any(int w, double (&acc)[LatGeo<WIN>::kNT + 1][2], int i0,
                                              int j0, int nj, double* Hc, double* bc) {
  if constexpr (W < LatGeo<WIN>::kNW) {
    if (w == W) lat_flush<WIN, W>(acc, i0, j0, nj, Hc, bc);
    else lat_flush_any<WIN, W + 1>(w, acc, i0, j0, nj, Hc, bc);
  }
}

template <int WIN>
__global__ void __launch_bounds__(32 * LatGeo<WIN>::kWarps, 2) k_gram_lattice(
    LatticeView L, const double* __restrict__ xs, const double* __restrict__ ys,
    const double* __restrict__ zs, const uint32_t* __restrict__ ms, const uint32_t* __restrict__ start,
    int nseg, int seg_len, double r2, double neg_inv_2b2, double scale, double* __restrict__ Hlat,
    double* __restrict__ blat) {
  using G = LatGeo<WIN>;
  constexpr int kB = G::kBatch;
  extern __shared__ __align__(16) unsigned char lat_smem[];
  double* Fbuf = reinterpret_cast<double*>(lat_smem);      // [2][kRows][kFP]
  double* sey = Fbuf + 2 * G::kRows * G::kFP;              // [warp][kPPW][WIN] e^{c dy^2}
  double* sdy2 = sey + G::kWarps * G::kPPW * WIN;          // dy^2, +inf outside the cell window
  uint32_t* need = reinterpret_cast<uint32_t*>(sdy2 + G::kWarps * G::kPPW * WIN);  // [WIN]
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int pl = lane / WIN, r = lane % WIN;  // this lane's point (in the warp) and window column
  const bool lane_on = pl < G::kPPW;
  const int ib = blockIdx.x / nseg, seg = blockIdx.x % nseg;
  const int i0 = ib - L.lo;
  if (i0 < 0 || i0 + WIN > L.ni) return;
  const int nj = L.nj;
  const size_t nn = static_cast<size_t>(L.ni) * nj;
  const int colour = (ib % WIN) + WIN * (seg & 1);
  double* Hc = Hlat + colour * nn * G::kKO;
  double* bc = blat + colour * nn;
  const int jb_end = min(nj, (seg + 1) * seg_len);
  double* wey = sey + (w * G::kPPW + (lane_on ? pl : 0)) * WIN;
  double* wdy2 = sdy2 + (w * G::kPPW + (lane_on ? pl : 0)) * WIN;
  double acc[G::kNT + 1][2];
  for (int jb = seg * seg_len; jb < jb_end; ++jb) {
    const size_t cell = static_cast<size_t>(ib) * nj + jb;
    const uint32_t p_beg = start[cell], p_end = start[cell + 1];
    if (p_beg == p_end) continue;
    const int j0 = jb - L.lo;
    __syncthreads();  // the previous cell's last products read F / need
    if (tid < WIN) {  // window column tid: nodes present, pair class not always-outside
      uint32_t bits = 0;
      const int* pc = L.P + (i0 + tid) * static_cast<size_t>(nj) + j0;
      for (int l = 0; l < WIN; ++l) bits |= (pc[l] != 0 ? 1u : 0u) << l;
      need[tid] = bits & (L.inmask[tid] | L.bdmask[tid]);
    }
#pragma unroll
    for (int t = 0; t <= G::kNT; ++t) acc[t][0] = acc[t][1] = 0.0;
    __syncthreads();
    const int nb = static_cast<int>((p_end - p_beg + kB - 1) / kB);
    // software pipeline: step b builds F block b (every warp, its own points:
    // the y factors, a __syncwarp, the row segments) while the DMMA warps
    // multiply F block b - 1; one barrier per block
    // this lane's point of the next batch, loaded one batch ahead
    const int p_lane = w * G::kPPW + pl;
    double nx = 0.0, ny = 0.0, nz = 0.0;
    uint32_t nm = 0;
    auto fetch_pt = [&](int bb) {
      const uint32_t pb = p_beg + static_cast<uint32_t>(bb) * kB;
      const int cnt = static_cast<int>(min(static_cast<uint32_t>(kB), p_end - pb));
      if (lane_on && p_lane < cnt) {
        nx = xs[pb + p_lane];
        ny = ys[pb + p_lane];
        nm = ms[pb + p_lane];
        if (r == 0) nz = zs[pb + p_lane];
      }
    };
    fetch_pt(0);
    for (int b = 0; b <= nb; ++b) {
      if (b < nb) {
        const uint32_t pb = p_beg + static_cast<uint32_t>(b) * kB;
        const int cnt = static_cast<int>(min(static_cast<uint32_t>(kB), p_end - pb));
        double* F = Fbuf + (b & 1) * G::kRows * G::kFP;
        const int p = p_lane;  // batch point of this lane
        const bool live = lane_on && p < cnt;
        const double px = nx, py = ny, pz = nz;
        const uint32_t msk = nm;
        if (b + 1 < nb) fetch_pt(b + 1);
        if (lane_on) {  // y factor of window row r for this point
          double e = 0.0, d2 = CUDART_INF;
          if (live) {
            const double d = __dsub_rn(__dadd_rn(L.min_y, __dmul_rn(static_cast<double>(j0 + r + L.j_org), L.res)), py);
            const double dd = __dmul_rn(d, d);
            if ((msk >> (16 + r)) & 1u) d2 = dd;
            e = exp(dd * neg_inv_2b2);
          }
          wey[r] = e;
          wdy2[r] = d2;
        }
        __syncwarp();
        if (lane_on && p < kB) {
          // F row segment (point p, window column r): always-inside pairs
          // unconditionally, boundary pairs with the reference's no-FMA
          // d^2 <= r^2 test (cell window folded into +inf), others zero
          double* row = F + p * G::kFP + r * WIN;
          if (live) {
            const double d = __dsub_rn(__dadd_rn(L.min_x, __dmul_rn(static_cast<double>(i0 + r + L.i_org), L.res)), px);
            const double dd = __dmul_rn(d, d);
            const double dx2 = ((msk >> r) & 1u) ? dd : CUDART_INF;
            const double ex = scale * exp(dd * neg_inv_2b2);
            const uint32_t nd = need[r], inm = L.inmask[r];
#pragma unroll
            for (int l = 0; l < WIN; ++l) {
              double v = 0.0;
              if ((nd >> l) & 1u)
                if (((inm >> l) & 1u) || __dadd_rn(dx2, wdy2[l]) <= r2) v = ex * wey[l];
              row[l] = v;
            }
            if (r == 0) row[G::kF] = pz;
          } else {
#pragma unroll
            for (int l = 0; l < WIN; ++l) row[l] = 0.0;
            if (r == 0) row[G::kF] = 0.0;
          }
          if (G::kF + 1 + r < G::kNT * 8) F[p * G::kFP + G::kF + 1 + r] = 0.0;
        }
        // rows beyond the batch (k-step padding) stay zero
        for (int q = kB * G::kFP + tid; q < G::kRows * G::kFP; q += 32 * G::kWarps) F[q] = 0.0;
        __syncwarp();
      }
      if (b > 0 && w < G::kNW) {
        const uint32_t pb = p_beg + static_cast<uint32_t>(b - 1) * kB;
        const int cnt = static_cast<int>(min(static_cast<uint32_t>(kB), p_end - pb));
        lat_mma_any<WIN>(w, Fbuf + ((b - 1) & 1) * G::kRows * G::kFP, (cnt + 3) >> 2, acc);
      }
      __syncthreads();
    }
    // the previous cell's adds to shared partners were ordered by the
    // barriers above (another thread may own the same entry this time)
    if (w < G::kNW) lat_flush_any<WIN>(w, acc, i0, j0, nj, Hc, bc);
  }
}

// H[max(ma, mb) + min(ma, mb) ld] += sum over colours (fixed order); b[ma] +=
// the colours' z rows.
__global__ void k_lat_reduce(const double* __restrict__ Hlat, const double* __restrict__ blat,
                             int ncol, int win, int ni, int nj, const int* __restrict__ nrow,
                             double* __restrict__ H, int ld, int band, double* __restrict__ b,
                             int* __restrict__ err) {
  const int ko = win * (2 * win - 1);
  const size_t nn = static_cast<size_t>(ni) * nj;
  const size_t total = nn * ko;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
       e += (size_t)gridDim.x * blockDim.x) {
    const size_t a = e / ko;
    const int k = static_cast<int>(e % ko);
    const int ma = nrow[a];
    if (ma < 0) continue;
    if (k == 0) {
      double s = 0.0;
      for (int c = 0; c < ncol; ++c) s += blat[c * nn + a];
      if (s != 0.0) b[ma] += s;
    }
    const int di = k / (2 * win - 1) - (win - 1), dj = k % (2 * win - 1) - (win - 1);
    if (di == 0 && dj > 0) continue;
    const int ia = static_cast<int>(a / nj), ja = static_cast<int>(a % nj);
    const int ip = ia + di, jp = ja + dj;
    if (ip < 0 || jp < 0 || jp >= nj) continue;
    const int mb = nrow[static_cast<size_t>(ip) * nj + jp];
    if (mb < 0) continue;
    double s = 0.0;
    for (int c = 0; c < ncol; ++c) s += Hlat[(c * nn + a) * ko + k];
    if (s == 0.0) continue;
    const int r = max(ma, mb), cc = min(ma, mb);
    if (r - cc > band) {
      atomicOr(err, 1);
      continue;
    }
    H[r + static_cast<size_t>(cc) * ld] += s;
  }
}

__global__ void k_lat_nrow(const int* __restrict__ slot, const int* __restrict__ rowof, int nc,
                           int* __restrict__ nrow) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < nc && rowof[c] >= 0) nrow[slot[c]] = rowof[c];
}

template <int WIN>
void launch_gram_lattice(tlg_ctx* ctx, const LatticeView& L, const double* xs, const double* ys,
                         const double* zs, const uint32_t* ms, const uint32_t* start, int nseg,
                         int seg_len, const KernelConst& kc, double* Hlat, double* blat) {
  using G = LatGeo<WIN>;
  TLG_CUDA(cudaFuncSetAttribute(k_gram_lattice<WIN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(G::kSmem)));
  k_gram_lattice<WIN><<<static_cast<unsigned>(L.ni) * nseg, 32 * G::kWarps, G::kSmem, ctx->stream>>>(
      L, xs, ys, zs, ms, start, nseg, seg_len, kc.r2, kc.neg_inv_2st2, kc.scale, Hlat, blat);
}

}  // namespace

// Lattice assembly of H (band storage, lower, ld; already holding lambda I or
// zero) += Mt Mt^T and b += Mt z over the mm observations (device x, y, z).
// rowof: centre id -> merged row. Returns false (nothing done) when the
// centres are not a lattice or the window is too wide for the tile kernel.
bool lattice_gram_device(tlg_model* m, const double* x, const double* y, const double* z,
                         size_t mm, const int* rowof, int band, double* H, int ld, double* b) {
  tlg_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  const LatticeGrid& LG = m->lat;
  m->last_gram_lattice = 0;
  if (!LG.valid || LG.win < 4 || LG.win > 12 || mm >= (1ull << 32)) return false;
  const int win = LG.win;
  const LatticeView L = lattice_view(m);
  const size_t nn = static_cast<size_t>(LG.ni) * LG.nj;
  // the per-cell blocks carry a fixed per-cell cost (the window Gram flush);
  // measured at C3 m = 20,000 (~5 observations per cell) they still beat the
  // row-wise CSR Gram (0.53 vs 0.63 ms), so only batches below ~2 per cell
  // keep the CSR path (env TLG_LAT_MIN_PER_CELL overrides)
  static const int min_per_cell = [] {
    const char* e = std::getenv("TLG_LAT_MIN_PER_CELL");
    return e ? std::atoi(e) : 2;
  }();
  if (mm < static_cast<size_t>(min_per_cell) * nn) return false;
  const int ko = win * (2 * win - 1);
  // column segments: >= 4 CTAs per SM in all, each >= WIN cells long (same-
  // parity segments of one column then never share a node window)
  int nseg = static_cast<int>(std::min<long long>((4ll * ctx->num_sms + LG.ni - 1) / LG.ni,
                                                  std::max(1, LG.nj / win)));
  nseg = std::max(1, nseg);
  const int seg_len = (LG.nj + nseg - 1) / nseg;
  const int ncol = nseg > 1 ? 2 * win : win;
  const size_t lat_elems = static_cast<size_t>(ncol) * nn * (ko + 1);
  if (lat_elems * 8 > (size_t{16} << 30)) return false;
  double* Hlat = ctx->ws<double>(S_LATGRAM, lat_elems);
  double* blat = Hlat + static_cast<size_t>(ncol) * nn * ko;
  TLG_CUDA(cudaMemsetAsync(Hlat, 0, lat_elems * 8, s));

  // cell order (stable: a fixed observation order per cell)
  uint32_t* key = ctx->ws<uint32_t>(S_KEYS, mm);
  uint32_t* key2 = ctx->ws<uint32_t>(S_KEYS2, mm);
  uint32_t* idx = ctx->ws<uint32_t>(S_VALS, mm);
  uint32_t* perm = ctx->ws<uint32_t>(S_VALS2, mm);
  const uint32_t skip = static_cast<uint32_t>(nn);
  k_lat_keys<<<static_cast<unsigned>((mm + 255) / 256), 256, 0, s>>>(L, win, x, y, mm, skip, key, idx);
  TLG_LAUNCHED(ctx);
  int end_bit = 1;
  while (end_bit < 32 && (1ull << end_bit) <= nn) ++end_bit;
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, key2, idx, perm, static_cast<int>(mm), 0, end_bit, s);
  void* dtmp = ctx->ws<unsigned char>(S_CUB, tmp);
  TLG_CUDA(cub::DeviceRadixSort::SortPairs(dtmp, tmp, key, key2, idx, perm, static_cast<int>(mm), 0,
                                           end_bit, s));
  ++ctx->launches;
  uint32_t* start = ctx->ws<uint32_t>(S_LATSTART, nn + 1);
  k_lat_bounds<<<static_cast<unsigned>((nn + 256) / 256), 256, 0, s>>>(key2, mm, static_cast<uint32_t>(nn), start);
  TLG_LAUNCHED(ctx);
  double* pts = ctx->ws<double>(S_LATPTS, 3 * mm + (mm + 1) / 2);
  uint32_t* msk = reinterpret_cast<uint32_t*>(pts + 3 * mm);
  k_lat_gather<<<static_cast<unsigned>((mm + 255) / 256), 256, 0, s>>>(
      L, win, perm, key2, skip, mm, x, y, z, pts, pts + mm, pts + 2 * mm, msk);
  TLG_LAUNCHED(ctx);

  switch (win) {
    case 4: launch_gram_lattice<4>(ctx, L, pts, pts + mm, pts + 2 * mm, msk, start, nseg, seg_len, m->kc, Hlat, blat); break;
    case 5: launch_gram_lattice<5>(ctx, L, pts, pts + mm, pts + 2 * mm, msk, start, nseg, seg_len, m->kc, Hlat, blat); break;
    case 6: launch_gram_lattice<6>(ctx, L, pts, pts + mm, pts + 2 * mm, msk, start, nseg, seg_len, m->kc, Hlat, blat); break;
    case 7: launch_gram_lattice<7>(ctx, L, pts, pts + mm, pts + 2 * mm, msk, start, nseg, seg_len, m->kc, Hlat, blat); break;
    case 8: launch_gram_lattice<8>(ctx, L, pts, pts + mm, pts + 2 * mm, msk, start, nseg, seg_len, m->kc, Hlat, blat); break;
    case 9: launch_gram_lattice<9>(ctx, L, pts, pts + mm, pts + 2 * mm, msk, start, nseg, seg_len, m->kc, Hlat, blat); break;
    case 10: launch_gram_lattice<10>(ctx, L, pts, pts + mm, pts + 2 * mm, msk, start, nseg, seg_len, m->kc, Hlat, blat); break;
    case 11: launch_gram_lattice<11>(ctx, L, pts, pts + mm, pts + 2 * mm, msk, start, nseg, seg_len, m->kc, Hlat, blat); break;
    default: launch_gram_lattice<12>(ctx, L, pts, pts + mm, pts + 2 * mm, msk, start, nseg, seg_len, m->kc, Hlat, blat); break;
  }
  TLG_LAUNCHED(ctx);

  const int nc = static_cast<int>(m->hcx.size());
  int* nrow = ctx->ws<int>(S_LATNROW, nn);
  TLG_CUDA(cudaMemsetAsync(nrow, 0xff, nn * sizeof(int), s));
  k_lat_nrow<<<(nc + 255) / 256, 256, 0, s>>>(LG.slot.p, rowof, nc, nrow);
  TLG_LAUNCHED(ctx);
  int* err = ctx->ws<int>(S_FLAGS, 4);
  TLG_CUDA(cudaMemsetAsync(err, 0, sizeof(int), s));
  const size_t total = nn * ko;
  k_lat_reduce<<<static_cast<unsigned>(std::min<size_t>((total + 255) / 256, 16ull * ctx->num_sms)), 256, 0, s>>>(
      Hlat, blat, ncol, win, LG.ni, LG.nj, nrow, H, ld, band, b, err);
  TLG_LAUNCHED(ctx);
  int h = 0;
  TLG_CUDA(cudaMemcpyAsync(&h, err, sizeof(int), cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
  if (h) throw Error(TLG_RUNTIME_ERROR, "batch ridge: lattice Gram entry outside the band");
  m->last_gram_lattice = 1;
  return true;
}

}  // namespace tlg
