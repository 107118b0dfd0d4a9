// K5-K8: TerrainModel::recursive_update (terrain_model.cpp:145-253) and
// fit_batch_ridge (:269-308) on the device.
//
// Host side keeps only the model *structure* (births, block/tile ids — the
// reference's integer bookkeeping); every floating-point step runs in a
// kernel:
//   K5  sparse moment matrix Mt as CSR over observations (ids bit-exact,
//       values s * kappa_sigma_tilde, dropping kappa == 0 like :193);
//   K6  Gram / Woodbury products on the sparse pattern;
//   K7  the solve, in one of two algebraically identical forms:
//       (W) one-shot Woodbury (m <= n): S = I + Mt^T Hinv0 Mt (m x m),
//           w1 = w0 + K S^-1 (z - Mt^T w0), diag blocks of
//           Hinv1 = Hinv0 - (L^-1 K^T)^T (L^-1 K^T);
//       (I) information form (m > n): H1 = blockdiag(info_inv)^-1 + Mt Mt^T,
//           w1 = w0 + H1^-1 Mt (z - Mt^T w0), diag blocks of H1^-1;
//       both equal the reference's chunk-64 Woodbury composition in exact
//       arithmetic (comment at :211-212); dense products use DMMA.
//   Re-split keeps only the active diagonal blocks, symmetrised (:239-251).
// A failed (non-PD) inner factorisation reports `rejected` and leaves
// weights/blocks untouched while births persist (:222-225).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>

#include "dense.cuh"
#include "dense_tile.cuh"

namespace tlg {

void block_resize(tlg_model* m, uint32_t b, int old_n, int new_n);
void upload_new_centres(tlg_model* m, size_t first);
uint32_t add_center_host(tlg_model* m, double x, double y);

// ---------------------------------------------------------------------------
// Neighbour sweep shared by the CSR builders (same cells/test as K3).
struct Sweep {
  int x_lo, x_hi, y_lo, y_hi;
};
__device__ __forceinline__ Sweep sweep_of(const GridView& g, double px, double py) {
  const int qx = static_cast<int>(floor(px / g.cell));
  const int qy = static_cast<int>(floor(py / g.cell));
  Sweep s;
  s.y_lo = max(qy - g.span - g.gy0, 0);
  s.y_hi = min(qy + g.span - g.gy0, g.gny - 1);
  s.x_lo = max(qx - g.span - g.gx0, 0);
  s.x_hi = min(qx + g.span - g.gx0, g.gnx - 1);
  if (s.y_lo > s.y_hi) s.x_hi = s.x_lo - 1;
  return s;
}

__global__ void k_mark_blocks(const uint8_t* __restrict__ active,
                              const uint32_t* __restrict__ bidx, size_t n,
                              uint8_t* __restrict__ bflag) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i < n && active[i]) bflag[bidx[i]] = 1;
}

__global__ void k_scatter_rowof(const uint32_t* __restrict__ merged, int n,
                                int* __restrict__ rowof) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) rowof[merged[r]] = r;
}

// CSR count / fill over observations: entry (col, s * exp(-d2/(2 b^2))) for
// every candidate with d2 <= cutoff^2 and kappa != 0. col = rowof[id] or id.
// Warp-per-observation variants (observation counts per scan are small, so
// one thread per observation walking ~190 candidates serially leaves the GPU
// idle): lanes stride over the candidate runs of the 3 cell columns; the fill
// keeps the serial candidate order through a ballot prefix.
__global__ void __launch_bounds__(128) k_mark_active_w(GridView g, const double* __restrict__ x,
                                                       const double* __restrict__ y, size_t m,
                                                       double r2, uint8_t* __restrict__ active) {
  const int lane = threadIdx.x & 31;
  const size_t nw = (size_t)gridDim.x * (blockDim.x >> 5);
  for (size_t i = blockIdx.x * (size_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < m; i += nw) {
    const double px = x[i], py = y[i];
    const Sweep s = sweep_of(g, px, py);
    for (int gx = s.x_lo; gx <= s.x_hi; ++gx) {
      const int b = g.cell_start[gx * g.gny + s.y_lo], e = g.cell_start[gx * g.gny + s.y_hi + 1];
      for (int k = b + lane; k < e; k += 32)
        if (sq2_exact(g.cx[k] - px, g.cy[k] - py) <= r2) {
          const uint32_t id = g.id[k];
          if (!active[id]) active[id] = 1;  // most ids are hit by many points
        }
    }
  }
}

__global__ void __launch_bounds__(128) k_csr_count_w(GridView g, const double* __restrict__ x,
                                                     const double* __restrict__ y, size_t m,
                                                     double r2, double neg_inv_2b2,
                                                     uint32_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const size_t nw = (size_t)gridDim.x * (blockDim.x >> 5);
  for (size_t i = blockIdx.x * (size_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < m; i += nw) {
    const double px = x[i], py = y[i];
    const Sweep s = sweep_of(g, px, py);
    uint32_t c = 0;
    for (int gx = s.x_lo; gx <= s.x_hi; ++gx) {
      const int b = g.cell_start[gx * g.gny + s.y_lo], e = g.cell_start[gx * g.gny + s.y_hi + 1];
      for (int k = b + lane; k < e; k += 32) {
        const double d2 = sq2_exact(g.cx[k] - px, g.cy[k] - py);
        if (d2 <= r2 && exp(d2 * neg_inv_2b2) != 0.0) ++c;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[i] = c;
  }
}

__global__ void __launch_bounds__(128) k_csr_fill_w(GridView g, const double* __restrict__ x,
                                                    const double* __restrict__ y, size_t m,
                                                    double r2, double neg_inv_2b2, double scale,
                                                    const uint32_t* __restrict__ rowp,
                                                    const int* __restrict__ rowof,
                                                    uint32_t* __restrict__ col,
                                                    double* __restrict__ val, int sort_ids) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const size_t nw = (size_t)gridDim.x * (blockDim.x >> 5);
  for (size_t i = blockIdx.x * (size_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < m; i += nw) {
    const double px = x[i], py = y[i];
    const Sweep s = sweep_of(g, px, py);
    uint32_t o = rowp[i];
    const uint32_t o0 = o;
    for (int gx = s.x_lo; gx <= s.x_hi; ++gx) {
      const int b = g.cell_start[gx * g.gny + s.y_lo], e = g.cell_start[gx * g.gny + s.y_hi + 1];
      for (int k0 = b; k0 < e; k0 += 32) {
        const int k = k0 + lane;
        bool take = false;
        double kv = 0.0;
        if (k < e) {
          const double d2 = sq2_exact(g.cx[k] - px, g.cy[k] - py);
          if (d2 <= r2) {
            kv = exp(d2 * neg_inv_2b2);
            take = kv != 0.0;
          }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, take);
        if (take) {
          const uint32_t pos = o + __popc(bal & lt);
          const uint32_t id = g.id[k];
          col[pos] = rowof ? static_cast<uint32_t>(rowof[id]) : id;
          val[pos] = scale * kv;
        }
        o += __popc(bal);
      }
    }
    __syncwarp();
    if (sort_ids && lane == 0)
      for (uint32_t a = o0 + 1; a < o; ++a) {
        const uint32_t ki = col[a];
        const double kvv = val[a];
        uint32_t b = a;
        while (b > o0 && col[b - 1] > ki) {
          col[b] = col[b - 1];
          val[b] = val[b - 1];
          --b;
        }
        col[b] = ki;
        val[b] = kvv;
      }
    __syncwarp();
  }
}

static unsigned warp_grid(size_t m, int num_sms) {
  return static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>((m + 3) / 4, 64ull * num_sms)));
}

struct Csr {
  uint32_t* rowp = nullptr;
  uint32_t* col = nullptr;
  double* val = nullptr;
  size_t nnz = 0;
};

// Builds the CSR in ctx slots (rowp may be supplied).
static Csr build_csr(tlg_model* m, const double* x, const double* y, size_t mm, const int* rowof,
                     double neg_inv_2b2, double scale, bool sort_ids, uint32_t* rowp_in) {
  tlg_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  Csr c;
  c.rowp = rowp_in ? rowp_in : ctx->ws<uint32_t>(S_ROWPTR, mm + 1);
  const GridView g = grid_view(m);
  k_csr_count_w<<<warp_grid(mm, ctx->num_sms), 128, 0, s>>>(g, x, y, mm, m->kc.r2, neg_inv_2b2, c.rowp);
  TLG_LAUNCHED(ctx);
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, c.rowp, c.rowp, (int)(mm + 1), s);
  void* dtmp = ctx->ws<unsigned char>(S_CUB, tmp);
  // the count array has mm entries; entry mm must be 0 before the scan
  TLG_CUDA(cudaMemsetAsync(c.rowp + mm, 0, sizeof(uint32_t), s));
  TLG_CUDA(cub::DeviceScan::ExclusiveSum(dtmp, tmp, c.rowp, c.rowp, (int)(mm + 1), s));
  ++ctx->launches;
  uint32_t hn = 0;
  TLG_CUDA(cudaMemcpyAsync(&hn, c.rowp + mm, 4, cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
  c.nnz = hn;
  c.col = ctx->ws<uint32_t>(S_COLIDX, hn + 1);
  c.val = ctx->ws<double>(S_MTVAL, hn + 1);
  k_csr_fill_w<<<warp_grid(mm, ctx->num_sms), 128, 0, s>>>(g, x, y, mm, m->kc.r2, neg_inv_2b2, scale, c.rowp, rowof, c.col,
                                c.val, sort_ids ? 1 : 0);
  TLG_LAUNCHED(ctx);
  return c;
}

void moment_device(tlg_model* m, const double* x, const double* y, size_t n, uint32_t* rowp,
                   uint32_t** ids, double** vals, size_t* nnz) {
  ensure_grid(m);
  tlg_ctx* ctx = m->ctx;
  // domain check (terrain_model.cpp:98)
  validate_obs_device(ctx, x, y, x, n, n);
  const Csr c = build_csr(m, x, y, n, nullptr, m->kc.neg_inv_2st2, m->kc.scale, true, rowp);
  *ids = c.col;
  *vals = c.val;
  *nnz = c.nnz;
}

// ---------------------------------------------------------------------------
// Merged-system bookkeeping.
struct BlockTab {  // per merged block q
  size_t pool_off;
  int ld;
  int n;        // n_q
  int off;      // first merged row
  int pad;
};

// r_j = z_j - m_j . w: a warp per observation (lanes over its entries,
// fixed shuffle tree)
__global__ void k_residual(const uint32_t* __restrict__ rowp, const uint32_t* __restrict__ col,
                           const double* __restrict__ val, const double* __restrict__ z,
                           const double* __restrict__ wm, size_t m, double* __restrict__ resid) {
  const size_t j = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= m) return;
  double s = 0.0;
  for (uint32_t e = rowp[j] + lane; e < rowp[j + 1]; e += 32) s = fma(val[e], wm[col[e]], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) resid[j] = z[j] - s;
}

__global__ void k_gather_w(const double* __restrict__ w, const uint32_t* __restrict__ merged, int n,
                           double* __restrict__ wm) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) wm[r] = w[merged[r]];
}

__global__ void k_apply_dw(double* __restrict__ w, const uint32_t* __restrict__ merged, int n,
                           const double* __restrict__ dw) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) w[merged[r]] += dw[r];
}

// Kt (m x n, ld m) = (Hinv0 Mt)^T ; one CTA per observation. Each (j, row)
// is only touched by one thread -> deterministic, no atomics.
__global__ void __launch_bounds__(128) k_build_Kt(
    const uint32_t* __restrict__ rowp, const uint32_t* __restrict__ col,
    const double* __restrict__ val, const int* __restrict__ rowblk,
    const int* __restrict__ rowloc, const BlockTab* __restrict__ tab,
    const double* __restrict__ pool, int m, double* __restrict__ Kt) {
  // Runs of consecutive entries in the same block (the candidate sweep visits
  // a block's centres together): per run each thread accumulates its rows
  // over the run's entries in a register and updates Kt once.
  const int j = blockIdx.x;
  const uint32_t e_end = rowp[j + 1];
  for (uint32_t e = rowp[j]; e < e_end;) {
    const int b = rowblk[col[e]];
    uint32_t f = e + 1;
    while (f < e_end && rowblk[col[f]] == b) ++f;
    const BlockTab t = tab[b];
    for (int i = threadIdx.x; i < t.n; i += blockDim.x) {
      double acc = 0.0;
      for (uint32_t q = e; q < f; ++q)
        acc = fma(pool[t.pool_off + static_cast<size_t>(rowloc[col[q]]) * t.ld + i], val[q], acc);
      Kt[j + static_cast<size_t>(t.off + i) * m] += acc;
    }
    e = f;
  }
}

// S = I + Mt^T K (m x m): CTA per row i, threads over columns j.
__global__ void __launch_bounds__(256) k_build_S(const uint32_t* __restrict__ rowp,
                                                 const uint32_t* __restrict__ col,
                                                 const double* __restrict__ val,
                                                 const double* __restrict__ Kt, int m,
                                                 double* __restrict__ S) {
  const int i = blockIdx.x;
  const uint32_t b = rowp[i], e = rowp[i + 1];
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    double s = 0.0;
    for (uint32_t q = b; q < e; ++q) s = fma(val[q], Kt[j + static_cast<size_t>(col[q]) * m], s);
    S[i + static_cast<size_t>(j) * m] = s + (i == j ? 1.0 : 0.0);
  }
}

// Symmetrise every merged block of the pool in place.
// A_q <- 0.5 (A_q + A_q^T) per block. Blocks that fit are staged through
// shared memory (one coalesced read and one coalesced write per element);
// larger ones are symmetrised in place in global memory.
__global__ void k_symmetrize_blocks_global(const BlockTab* __restrict__ tab,
                                           double* __restrict__ pool) {
  const BlockTab t = tab[blockIdx.x];
  double* a = pool + t.pool_off;
  for (int e = threadIdx.x; e < t.n * t.n; e += blockDim.x) {
    const int r = e % t.n, c = e / t.n;
    if (r > c) {
      const double v = 0.5 * (a[r + (size_t)c * t.ld] + a[c + (size_t)r * t.ld]);
      a[r + (size_t)c * t.ld] = v;
      a[c + (size_t)r * t.ld] = v;
    }
  }
}

__global__ void k_symmetrize_blocks(const BlockTab* __restrict__ tab, double* __restrict__ pool) {
  extern __shared__ double sb[];
  const BlockTab t = tab[blockIdx.x];
  double* a = pool + t.pool_off;
  const int nn = t.n * t.n;
  for (int e = threadIdx.x; e < nn; e += blockDim.x) sb[e] = a[(e % t.n) + (size_t)(e / t.n) * t.ld];
  __syncthreads();
  for (int e = threadIdx.x; e < nn; e += blockDim.x) {
    const int r = e % t.n, c = e / t.n;
    const double v = r == c ? sb[e] : 0.5 * (r > c ? sb[e] + sb[c + r * t.n] : sb[c + r * t.n] + sb[e]);
    a[r + (size_t)c * t.ld] = v;
  }
}

// Transposed CSR (rows of Mt): bucket entries by row, j ascending.
__global__ void k_expand_rows(const uint32_t* __restrict__ rowp, size_t m,
                              uint32_t* __restrict__ obs_of) {
  const size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  for (uint32_t e = rowp[j]; e < rowp[j + 1]; ++e) obs_of[e] = static_cast<uint32_t>(j);
}

__global__ void k_row_hist(const uint32_t* __restrict__ col, size_t nnz, uint32_t* __restrict__ cnt) {
  const size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (e < nnz) atomicAdd(&cnt[col[e]], 1u);
}

// Few rows, many entries (C1: 256 rows, 1.2M entries): privatised counts in
// shared memory, then one global add per nonzero bin and block.
__global__ void k_row_hist_smem(const uint32_t* __restrict__ col, size_t nnz, int n,
                                uint32_t* __restrict__ cnt) {
  extern __shared__ uint32_t hb[];
  for (int r = threadIdx.x; r < n; r += blockDim.x) hb[r] = 0;
  __syncthreads();
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < nnz;
       e += (size_t)gridDim.x * blockDim.x)
    atomicAdd(&hb[col[e]], 1u);
  __syncthreads();
  for (int r = threadIdx.x; r < n; r += blockDim.x)
    if (hb[r]) atomicAdd(&cnt[r], hb[r]);
}

// Gram row r: G[r, :] = sum_{j in row r} v_rj * Mt[:, j]; shared-memory row
// accumulator, observations in ascending order -> deterministic. Adds into
// column r of H (H symmetric, col-major) so writes are coalesced.
__global__ void __launch_bounds__(128) k_gram_rows(
    const uint32_t* __restrict__ trowp, const uint32_t* __restrict__ tobs,
    const double* __restrict__ tval, const uint32_t* __restrict__ rowp,
    const uint32_t* __restrict__ col, const double* __restrict__ val, int n,
    double* __restrict__ H, int ldh) {
  extern __shared__ double acc[];
  const int r = blockIdx.x;
  for (int s = threadIdx.x; s < n; s += blockDim.x) acc[s] = 0.0;
  __syncthreads();
  for (uint32_t q = trowp[r]; q < trowp[r + 1]; ++q) {
    const uint32_t j = tobs[q];
    const double vr = tval[q];
    for (uint32_t e = rowp[j] + threadIdx.x; e < rowp[j + 1]; e += blockDim.x)
      acc[col[e]] = fma(vr, val[e], acc[col[e]]);
    __syncthreads();
  }
  for (int s = threadIdx.x; s < n; s += blockDim.x) H[s + (size_t)r * ldh] += acc[s];
}

// Transposed CSR of Mt (by merged row).
struct TCsr {
  uint32_t* rowp;
  uint32_t* obs;
  double* val;
};

// Banded Gram: one warp per (row r, observation chunk c) accumulates that
// chunk's part of row r of Mt Mt^T over the columns [r - band, r + band] in a
// per-warp shared window (observations in ascending order, an observation's
// entries have distinct columns -> no races, deterministic). With one chunk
// per row the window is added into column r of H; with nch > 1 (few rows,
// many observations per row: the C1 regime) each chunk's window goes to
// partials[c][r][:] and k_gram_chunks_reduce sums the chunks in order.
constexpr int kGramWarps = 4;
__global__ void __launch_bounds__(32 * kGramWarps) k_gram_rows_band(
    const uint32_t* __restrict__ trowp, const uint32_t* __restrict__ tobs,
    const double* __restrict__ tval, const uint32_t* __restrict__ rowp,
    const uint32_t* __restrict__ col, const double* __restrict__ val, int n, int band,
    int lower_only, double* __restrict__ H, int ldh, int nch, double* __restrict__ partials) {
  extern __shared__ double gsm[];
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  // lower_only: row r accumulates only columns >= r (band storage of the
  // lower triangle; the symmetric half is neither computed nor written)
  const int width = lower_only ? band + 1 : 2 * band + 1;
  double* acc = gsm + wq * width;
  const long long items = static_cast<long long>(n) * nch;
  for (long long it = blockIdx.x * (long long)kGramWarps + wq; it < items;
       it += (long long)gridDim.x * kGramWarps) {
    const int r = static_cast<int>(it / nch), ch = static_cast<int>(it % nch);
    const int lo = lower_only ? r : r - band;
    for (int s = lane; s < width; s += 32) acc[s] = 0.0;
    __syncwarp();
    const uint32_t rb = trowp[r], rn = trowp[r + 1] - rb;
    const uint32_t q_end = rb + static_cast<uint32_t>((static_cast<unsigned long long>(rn) * (ch + 1)) / nch);
    for (uint32_t q0 = rb + static_cast<uint32_t>((static_cast<unsigned long long>(rn) * ch) / nch);
         q0 < q_end; q0 += 32) {
      // lane-parallel fetch of 32 observations' metadata (one latency)
      const uint32_t qq = q0 + lane;
      uint32_t jb = 0, je = 0;
      double vr = 0.0;
      if (qq < q_end) {
        const uint32_t j = tobs[qq];
        vr = tval[qq];
        jb = rowp[j];
        je = rowp[j + 1];
      }
      const int cnt = static_cast<int>(min(32u, q_end - q0));
      // software pipeline: the entries of observations k + 1 .. k + kDepth
      // are in flight while k updates (a register ring, statically indexed)
      constexpr int kPre = 3;    // entries per lane and observation (96 per obs)
      constexpr int kDepth = 4;  // observations in flight
      int pc[kDepth][kPre];
      double pv[kDepth][kPre];
      auto fetch = [&](int k, int slot_c[kPre], double slot_v[kPre]) {
        const uint32_t b = __shfl_sync(0xffffffffu, jb, k & 31), e = __shfl_sync(0xffffffffu, je, k & 31);
#pragma unroll
        for (int u = 0; u < kPre; ++u) {
          const uint32_t x = b + lane + 32 * u;
          const bool ok = k < cnt && x < e;
          slot_c[u] = ok ? static_cast<int>(col[x]) - lo : -1;
          slot_v[u] = ok ? val[x] : 0.0;
        }
      };
#pragma unroll
      for (int d = 0; d < kDepth; ++d) fetch(d, pc[d], pv[d]);
      for (int k0 = 0; k0 < cnt; k0 += kDepth) {
#pragma unroll
        for (int d = 0; d < kDepth; ++d) {
          const int k = k0 + d;
          if (k < cnt) {  // warp-uniform
            int cc[kPre];
            double cv[kPre];
#pragma unroll
            for (int u = 0; u < kPre; ++u) {
              cc[u] = pc[d][u];
              cv[u] = pv[d][u];
            }
            const double v = __shfl_sync(0xffffffffu, vr, k);
            const uint32_t b = __shfl_sync(0xffffffffu, jb, k), e = __shfl_sync(0xffffffffu, je, k);
            fetch(k + kDepth, pc[d], pv[d]);
#pragma unroll
            for (int u = 0; u < kPre; ++u)
              if (cc[u] >= 0) acc[cc[u]] = fma(v, cv[u], acc[cc[u]]);
            // observations with more than 32 * kPre entries (other geometries)
            for (uint32_t x = b + 32 * kPre + lane; x < e; x += 32) {
              const int ci = static_cast<int>(col[x]) - lo;
              if (ci >= 0) acc[ci] = fma(v, val[x], acc[ci]);
            }
            __syncwarp();
          }
        }
      }
    }
    const int c0 = max(lo, 0), c1 = min(r + band, n - 1);  // H[c][r]: column r, c >= lo
    if (nch == 1) {
      for (int cc = c0 + lane; cc <= c1; cc += 32) H[cc + (size_t)r * ldh] += acc[cc - lo];
    } else {
      double* pr = partials + (static_cast<size_t>(ch) * n + r) * width;
      for (int cc = c0 + lane; cc <= c1; cc += 32) pr[cc - lo] = acc[cc - lo];
    }
    __syncwarp();
  }
}

// Chunk partials of the banded Gram summed in chunk order into H.
__global__ void k_gram_chunks_reduce(const double* __restrict__ partials, int n, int band,
                                     int lower_only, int nch, double* __restrict__ H, int ldh) {
  const int width = lower_only ? band + 1 : 2 * band + 1;
  const long long tot = static_cast<long long>(n) * width;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(e / width), s = static_cast<int>(e % width);
    const int lo = lower_only ? r : r - band;
    const int cc = lo + s;
    if (cc < 0 || cc >= n || cc > r + band) continue;
    double v = 0.0;
    for (int ch = 0; ch < nch; ++ch) v += partials[(static_cast<size_t>(ch) * n + r) * width + s];
    H[cc + static_cast<size_t>(r) * ldh] += v;
  }
}

static void gram_band(tlg_ctx* ctx, const TCsr& t, const Csr& c, int n, int band, double* H,
                      int ldh, bool lower_only = false) {
  const size_t width = lower_only ? band + 1 : 2 * static_cast<size_t>(band) + 1;
  const size_t smem_band = sizeof(double) * kGramWarps * width;
  if (smem_band <= 200 * 1024) {
    if (smem_band > 48 * 1024)
      TLG_CUDA(cudaFuncSetAttribute(k_gram_rows_band, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem_band));
    // observation chunks per row: enough warps to fill the GPU when rows are
    // few and long (~128 observations per chunk), within a partials budget
    const double obs_per_row = n ? static_cast<double>(c.nnz) / n : 0.0;
    int nch = static_cast<int>(std::min(obs_per_row / 256.0,
                                        (1.0 * ctx->num_sms * 8 * kGramWarps) / std::max(n, 1)));
    const size_t per_chunk = static_cast<size_t>(n) * width * sizeof(double);
    nch = std::max(1, std::min<int>(nch, static_cast<int>((256u << 20) / std::max<size_t>(per_chunk, 1))));
    double* partials = nch > 1 ? ctx->ws<double>(S_GRAMPART, static_cast<size_t>(nch) * n * width) : nullptr;
    const long long items = static_cast<long long>(n) * nch;
    const unsigned blocks = static_cast<unsigned>(
        std::min<long long>((items + kGramWarps - 1) / kGramWarps, 1ll << 20));
    k_gram_rows_band<<<blocks, 32 * kGramWarps, smem_band, ctx->stream>>>(
        t.rowp, t.obs, t.val, c.rowp, c.col, c.val, n, band, lower_only ? 1 : 0, H, ldh, nch,
        partials);
    if (nch > 1) {
      TLG_LAUNCHED(ctx);
      const long long tot = static_cast<long long>(n) * width;
      k_gram_chunks_reduce<<<static_cast<unsigned>(std::min<long long>((tot + 255) / 256, 8ull * ctx->num_sms)), 256, 0,
                             ctx->stream>>>(partials, n, band, lower_only ? 1 : 0, nch, H, ldh);
    }
  } else {
    require(!lower_only, TLG_RUNTIME_ERROR, "banded Gram: band too wide for band storage");
    const size_t smem = static_cast<size_t>(n) * 8;
    if (smem > 48 * 1024)
      TLG_CUDA(cudaFuncSetAttribute(k_gram_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_gram_rows<<<n, 128, smem, ctx->stream>>>(t.rowp, t.obs, t.val, c.rowp, c.col, c.val, n, H, ldh);
  }
  TLG_LAUNCHED(ctx);
}

// rhs b[r] = sum_{j in row r} v_rj * c_j  (c = residual or z)
// One warp per row: lane l sums entries l, l + 32, ... in order, then a
// fixed xor tree (deterministic; rows of thousands of entries in the C1
// regime no longer run on a single thread).
__global__ void k_row_dot(const uint32_t* __restrict__ trowp, const uint32_t* __restrict__ tobs,
                          const double* __restrict__ tval, const double* __restrict__ c, int n,
                          double* __restrict__ b) {
  const int lane = threadIdx.x & 31;
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n) return;
  double s = 0.0;
  for (uint32_t q = trowp[r] + lane; q < trowp[r + 1]; q += 32) s = fma(tval[q], c[tobs[q]], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) b[r] = s;
}

__global__ void k_copy_to_pool_blocks(const BlockTab* __restrict__ tab, const double* __restrict__ H,
                                      int ldh, double* __restrict__ pool) {
  const BlockTab t = tab[blockIdx.x];
  for (int e = threadIdx.x; e < t.n * t.n; e += blockDim.x) {
    const int r = e % t.n, c = e / t.n;
    pool[t.pool_off + r + (size_t)c * t.ld] = H[(t.off + r) + (size_t)(t.off + c) * ldh];
  }
}

__global__ void k_set_identity(double* __restrict__ X, int n, int ld) {
  const long long tot = (long long)n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(e % n), c = static_cast<int>(e / n);
    X[r + (size_t)c * ld] = (r == c) ? 1.0 : 0.0;
  }
}

__global__ void k_diag_minmax(const double* __restrict__ L, int n, int ld, double* __restrict__ out) {
  double mx = 0.0, mn = INFINITY;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = L[i + (size_t)i * ld];
    const double v = d * d;
    mx = fmax(mx, fabs(v));
    mn = fmin(mn, fabs(v));
  }
  __shared__ double smx[256], smn[256];
  smx[threadIdx.x] = mx;
  smn[threadIdx.x] = mn;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)blockDim.x; ++i) {
      mx = fmax(mx, smx[i]);
      mn = fmin(mn, smn[i]);
    }
    out[0] = mx;
    out[1] = mn;
  }
}

// SPD inverse of the n x n matrix src (lds) into dst (ldd) via Cholesky:
// the factorisation also yields X = L^-1, and A^-1 = X^T X is one GEMM.
static bool spd_inverse(tlg_ctx* ctx, const double* src, int lds, int n, double* dst, int ldd) {
  double* T = ctx->ws<double>(S_WORK2, static_cast<size_t>(n) * n);
  double* X = ctx->ws<double>(S_XINV2, static_cast<size_t>(n) * n);
  int* info = ctx->ws<int>(S_FLAGS, 4) + 1;
  TLG_CUDA(cudaMemsetAsync(info, 0, sizeof(int), ctx->stream));
  TLG_CUDA(cudaMemcpy2DAsync(T, n * 8, src, lds * 8, n * 8, n, cudaMemcpyDeviceToDevice, ctx->stream));
  potrf_lower(ctx, T, n, n, info, X, n);
  gemm(ctx, GemmDesc{n, n, n, X, n, 1, X, n, 0, dst, ldd, 1.0, 0.0, 0});
  int h = 0;
  TLG_CUDA(cudaMemcpyAsync(&h, info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  TLG_CUDA(cudaStreamSynchronize(ctx->stream));
  symmetrize(ctx, dst, n, ldd);
  return h == 0;
}

// All active blocks at once: one CTA per block q inverts info_inv_q (SPD,
// n_q <= kBatchInvMax) in shared memory with 32-wide tiles — per tile column
// k the diagonal tile is factored and inverted by one warp in registers
// (warp_potrf_inv32, dense_tile.cuh), the panel becomes a product with that
// inverse and the trailing triangle a rank-32 update; then X = L^-1 tile row
// by tile row (X_ij = -Linv_ii sum_m L_im X_mj), and A^-1 = X^T X is written
// into the diagonal block of H (ld ldd). ~6 barriers per tile instead of 5 per
// column; info != 0 on a non-positive pivot.
constexpr int kBatchInvMax = 112;
constexpr int kInvThreads = 256;
struct InvJob {  // dst (ldd) <- src(lds)^-1, n x n SPD
  const double* src;
  double* dst;
  int lds, ldd, n, pad;
};
__global__ void __launch_bounds__(kInvThreads) k_batched_spd_inverse(const InvJob* __restrict__ jobs,
                                                                     int* __restrict__ info) {
  extern __shared__ double sm[];
  const InvJob b = jobs[blockIdx.x];
  const int n = b.n, P = n + 1, t = threadIdx.x, lane = t & 31, wq = t >> 5;
  constexpr int nw = kInvThreads / 32;
  double* a = sm;                 // a[r + c P]: lower triangle -> L
  double* x = a + n * P;          // x[r + c P]: X = L^-1 (lower)
  double* linv = x + n * P;       // 32 x 32, ld 32
  double* scratch = linv + 32 * 32;
  const double* src = b.src;
  for (int e = t; e < n * n; e += kInvThreads) {
    const int r = e % n, c = e / n;
    a[r + c * P] = (r >= c) ? src[r + (size_t)c * b.lds] : 0.0;
    x[r + c * P] = 0.0;
  }
  __syncthreads();
  const int nt = (n + 31) / 32;
  for (int k = 0; k < nt; ++k) {
    const int k0 = 32 * k, kb = min(32, n - k0), r0 = k0 + kb;
    if (wq == 0) warp_potrf_inv32(a + k0 + k0 * P, P, kb, linv, info, scratch);
    __syncthreads();
    // X_kk = Linv_kk
    for (int e = t; e < kb * kb; e += kInvThreads) {
      const int r = e % kb, c = e / kb;
      x[k0 + r + (k0 + c) * P] = linv[r + c * 32];
    }
    // panel rows r >= r0: L[r][k0 + c] = sum_p A[r][k0 + p] Linv[c][p]
    for (int r = r0 + wq; r < n; r += nw) {
      double v = 0.0;
      if (lane < kb)
        for (int p = 0; p <= lane; ++p) v = fma(a[r + (k0 + p) * P], linv[lane + p * 32], v);
      __syncwarp();
      if (lane < kb) a[r + (k0 + lane) * P] = v;
    }
    __syncthreads();
    // trailing lower triangle: A[r][c] -= sum_p L[r][k0 + p] L[c][k0 + p]
    const int m = n - r0;
    for (int e = t; e < m * m; e += kInvThreads) {
      const int r = r0 + e % m, c = r0 + e / m;
      if (r < c) continue;
      double v = a[r + c * P];
      for (int p = 0; p < kb; ++p) v = fma(-a[r + (k0 + p) * P], a[c + (k0 + p) * P], v);
      a[r + c * P] = v;
    }
    __syncthreads();
  }
  // X = L^-1 below the diagonal tiles, tile row i ascending:
  // T = sum_{m=j}^{i-1} L_im X_mj (cols of tile column j), X_ij = -Linv_ii T
  for (int i = 1; i < nt; ++i) {
    const int i0 = 32 * i, ib = min(32, n - i0);
    // T into x's (i, j) tiles (currently zero), j < i
    for (int e = t; e < ib * i0; e += kInvThreads) {
      const int r = i0 + e % ib, c = e / ib;  // c < i0
      double v = 0.0;
      for (int q = c; q < i0; ++q) v = fma(a[r + q * P], x[q + c * P], v);
      x[r + c * P] = v;
    }
    __syncthreads();
    // X_ij = -Linv_ii T: Linv_ii is x's diagonal tile (i, i); column-wise in place
    for (int c = wq; c < i0; c += nw) {
      double v = 0.0;
      if (lane < ib)
        for (int q = 0; q <= lane; ++q) v = fma(x[i0 + lane + (i0 + q) * P], x[i0 + q + c * P], v);
      __syncwarp();
      if (lane < ib) x[i0 + lane + c * P] = -v;
    }
    __syncthreads();
  }
  // A^-1 = X^T X: (r, c) = sum_{p >= max(r, c)} x_pr x_pc; write both halves
  double* dst = b.dst;
  const int ldh = b.ldd;
  for (int e = t; e < n * n; e += kInvThreads) {
    const int r = e % n, c = e / n;
    if (r < c) continue;
    double s0 = 0.0, s1 = 0.0;
    int p = r;
    for (; p + 1 < n; p += 2) {
      s0 = fma(x[p + r * P], x[p + c * P], s0);
      s1 = fma(x[p + 1 + r * P], x[p + 1 + c * P], s1);
    }
    if (p < n) s0 = fma(x[p + r * P], x[p + c * P], s0);
    const double v = s0 + s1;
    dst[r + (size_t)c * ldh] = v;
    dst[c + (size_t)r * ldh] = v;
  }
}

// Launches k_batched_spd_inverse over host-built jobs (all n <= kBatchInvMax).
static void batched_spd_inverse(tlg_ctx* ctx, const std::vector<InvJob>& jobs, int* info) {
  if (jobs.empty()) return;
  int maxn = 0;
  for (const auto& j : jobs) maxn = std::max(maxn, j.n);
  const size_t bytes = jobs.size() * sizeof(InvJob);
  InvJob* h = static_cast<InvJob*>(ctx->host_stage(bytes));
  std::memcpy(h, jobs.data(), bytes);
  InvJob* d = reinterpret_cast<InvJob*>(ctx->ws<char>(S_BLKTAB, bytes));
  TLG_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, ctx->stream));
  const int smem = (2 * maxn * (maxn + 1) + 32 * 32 + kWarpPotrfSmem) * 8;
  TLG_CUDA(cudaFuncSetAttribute(k_batched_spd_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem));
  k_batched_spd_inverse<<<static_cast<unsigned>(jobs.size()), kInvThreads, smem, ctx->stream>>>(d, info);
  TLG_LAUNCHED(ctx);
}

__global__ void k_iota(uint32_t* __restrict__ a, size_t n) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = static_cast<uint32_t>(i);
}
static void iota_u32(tlg_ctx* ctx, uint32_t* a, size_t n) {
  k_iota<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(a, n);
  TLG_LAUNCHED(ctx);
}
__global__ void k_gather_tcsr(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ obs_of,
                              const double* __restrict__ val, size_t nnz, uint32_t* __restrict__ tobs,
                              double* __restrict__ tval) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= nnz) return;
  const uint32_t e = perm[i];
  tobs[i] = obs_of[e];
  tval[i] = val[e];
}
static void gather_tcsr(tlg_ctx* ctx, const uint32_t* perm, const uint32_t* obs_of, const double* val,
                 size_t nnz, uint32_t* tobs, double* tval) {
  k_gather_tcsr<<<(unsigned)((nnz + 255) / 256), 256, 0, ctx->stream>>>(perm, obs_of, val, nnz, tobs, tval);
  TLG_LAUNCHED(ctx);
}

// Transposed CSR of Mt (by merged row): trowp (n+1), tobs, tval.
static TCsr transpose_csr(tlg_ctx* ctx, const Csr& c, size_t m, int n) {
  cudaStream_t s = ctx->stream;
  TCsr t;
  t.rowp = ctx->ws<uint32_t>(S_TROWP, n + 1);
  uint32_t* obs_of = ctx->ws<uint32_t>(S_KEYS, c.nnz + 1);
  uint32_t* col_sorted = ctx->ws<uint32_t>(S_KEYS2, c.nnz + 1);
  t.obs = ctx->ws<uint32_t>(S_VALS, c.nnz + 1);
  t.val = ctx->ws<double>(S_U, c.nnz + 1);
  if (c.nnz) {
    k_expand_rows<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(c.rowp, m, obs_of);
    TLG_LAUNCHED(ctx);
  }
  TLG_CUDA(cudaMemsetAsync(t.rowp, 0, (n + 1) * sizeof(uint32_t), s));
  if (c.nnz) {
    if (n <= 12288) {
      const unsigned b = static_cast<unsigned>(std::min<size_t>((c.nnz + 1023) / 1024, 2ull * ctx->num_sms));
      k_row_hist_smem<<<b, 256, n * sizeof(uint32_t), s>>>(c.col, c.nnz, n, t.rowp);
    } else {
      k_row_hist<<<(unsigned)((c.nnz + 255) / 256), 256, 0, s>>>(c.col, c.nnz, t.rowp);
    }
    TLG_LAUNCHED(ctx);
  }
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, t.rowp, t.rowp, n + 1, s);
  void* dtmp = ctx->ws<unsigned char>(S_CUB, tmp);
  TLG_CUDA(cub::DeviceScan::ExclusiveSum(dtmp, tmp, t.rowp, t.rowp, n + 1, s));
  ++ctx->launches;
  if (c.nnz) {
    // stable sort of entry index by row keeps observations ascending per row
    uint32_t* eidx = ctx->ws<uint32_t>(S_VALS2, c.nnz + 1);
    uint32_t* eidx_sorted = ctx->ws<uint32_t>(S_NODE_IDX, c.nnz + 1);
    TLG_CUDA(cudaMemcpyAsync(col_sorted, c.col, c.nnz * 4, cudaMemcpyDeviceToDevice, s));
    tmp = 0;
    int end_bit = 1;
    while (end_bit < 32 && (1u << end_bit) < static_cast<uint32_t>(n)) ++end_bit;
    iota_u32(ctx, eidx, c.nnz);
    uint32_t* keys_out = ctx->ws<uint32_t>(S_TKEYS, c.nnz + 1);
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, col_sorted, keys_out, eidx, eidx_sorted,
                                    (int)c.nnz, 0, end_bit, s);
    dtmp = ctx->ws<unsigned char>(S_CUB2, tmp);
    TLG_CUDA(cub::DeviceRadixSort::SortPairs(dtmp, tmp, col_sorted, keys_out, eidx, eidx_sorted,
                                             (int)c.nnz, 0, end_bit, s));
    ++ctx->launches;
    gather_tcsr(ctx, eidx_sorted, obs_of, c.val, c.nnz, t.obs, t.val);
  }
  return t;
}

// ---------------------------------------------------------------------------
// Stage timer for diagnosis (env TLG_TRACE=1): synchronises and prints the
// wall time of each update stage to stderr. Off by default (no syncs).
struct StageTrace {
  tlg_ctx* ctx;
  bool on;
  std::chrono::steady_clock::time_point t0, last;
  std::string out;
  explicit StageTrace(tlg_ctx* c) : ctx(c), on(std::getenv("TLG_TRACE") != nullptr) {
    t0 = last = std::chrono::steady_clock::now();
  }
  void mark(const char* name) {
    if (!on) return;
    cudaStreamSynchronize(ctx->stream);
    const auto now = std::chrono::steady_clock::now();
    out += std::string(name) + "=" +
           std::to_string(std::chrono::duration<double, std::micro>(now - last).count()) + "us ";
    last = now;
  }
  ~StageTrace() {
    if (on)
      std::fprintf(stderr, "[tlg update] %s total=%.1fus\n", out.c_str(),
                   std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
  }
};

// Row-by-row order of blocks over the tile grid (the shorter extent fastest):
// with it, H = H0 + Mt Mt^T, which couples only blocks whose tiles touch
// (shared observations lie within the cutoff of both centres, tile side =
// 2 cutoff), is block-banded. Returns the tile coordinates per block id
// (empty when the model has a single tile).
static std::vector<std::pair<int64_t, int64_t>> spatial_block_order(
    const tlg_model* m, std::vector<uint32_t>& blocks) {
  std::vector<std::pair<int64_t, int64_t>> btile;
  if (m->tile_blocks.size() <= 1) return btile;
  btile.assign(m->members.size(), {0, 0});
  for (const auto& [key, b] : m->tile_blocks)
    btile[b] = {static_cast<int32_t>(static_cast<uint64_t>(key) >> 32),
                static_cast<int32_t>(static_cast<uint64_t>(key) & 0xffffffffu)};
  int64_t x0 = INT64_MAX, x1 = INT64_MIN, y0 = INT64_MAX, y1 = INT64_MIN;
  for (uint32_t b : blocks) {
    x0 = std::min(x0, btile[b].first);
    x1 = std::max(x1, btile[b].first);
    y0 = std::min(y0, btile[b].second);
    y1 = std::max(y1, btile[b].second);
  }
  const bool x_fast = (x1 - x0) <= (y1 - y0);
  auto key = [&](uint32_t b) {
    return x_fast ? std::make_pair(btile[b].second, btile[b].first)
                  : std::make_pair(btile[b].first, btile[b].second);
  };
  std::stable_sort(blocks.begin(), blocks.end(),
                   [&](uint32_t a, uint32_t b) { return key(a) < key(b); });
  return btile;
}

// Lower bandwidth (rows) of H under the merged order: a row of block q has no
// entry left of the first row of the earliest block whose tile touches q's.
static int block_band(const std::vector<std::pair<int64_t, int64_t>>& btile,
                      const std::vector<uint32_t>& blocks, const std::vector<BlockTab>& tab) {
  int band = 0;
  for (size_t q = 0; q < blocks.size(); ++q) {
    int first = tab[q].off;
    const auto& b = btile[blocks[q]];
    for (size_t p = 0; p < q; ++p) {
      const auto& a = btile[blocks[p]];
      if (std::llabs(a.first - b.first) <= 1 && std::llabs(a.second - b.second) <= 1) {
        first = tab[p].off;
        break;
      }
    }
    band = std::max(band, tab[q].off + tab[q].n - 1 - first);
  }
  return band;
}

// Births pre-check (steady state): a node can be born only if it is
// supported, and every supported node lies within r_a of a point, i.e. in
// the node window of the scan's bounding box dilated by r_a. If every node of
// that window already holds a centre (lattice presence > 0 implies the
// reference's occupancy key), nothing can be born and the support count is
// skipped. One CTA; out = 1 when some window node is unoccupied.
__global__ void __launch_bounds__(1024) k_births_precheck(
    const double* __restrict__ x, const double* __restrict__ y, size_t m, double min_x,
    double min_y, double res, double r_a, int nx, int ny, const int* __restrict__ P, int ni,
    int nj, int i_org, int j_org, int* __restrict__ out) {
  __shared__ double red[4][32];
  double lo_x = INFINITY, lo_y = INFINITY, hi_x = -INFINITY, hi_y = -INFINITY;
  for (size_t k = threadIdx.x; k < m; k += blockDim.x) {
    lo_x = fmin(lo_x, x[k]);
    hi_x = fmax(hi_x, x[k]);
    lo_y = fmin(lo_y, y[k]);
    hi_y = fmax(hi_y, y[k]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo_x = fmin(lo_x, __shfl_xor_sync(0xffffffffu, lo_x, o));
    hi_x = fmax(hi_x, __shfl_xor_sync(0xffffffffu, hi_x, o));
    lo_y = fmin(lo_y, __shfl_xor_sync(0xffffffffu, lo_y, o));
    hi_y = fmax(hi_y, __shfl_xor_sync(0xffffffffu, hi_y, o));
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red[0][w] = lo_x;
    red[1][w] = hi_x;
    red[2][w] = lo_y;
    red[3][w] = hi_y;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    lo_x = lane < nw ? red[0][lane] : INFINITY;
    hi_x = lane < nw ? red[1][lane] : -INFINITY;
    lo_y = lane < nw ? red[2][lane] : INFINITY;
    hi_y = lane < nw ? red[3][lane] : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo_x = fmin(lo_x, __shfl_xor_sync(0xffffffffu, lo_x, o));
      hi_x = fmax(hi_x, __shfl_xor_sync(0xffffffffu, hi_x, o));
      lo_y = fmin(lo_y, __shfl_xor_sync(0xffffffffu, lo_y, o));
      hi_y = fmax(hi_y, __shfl_xor_sync(0xffffffffu, hi_y, o));
    }
    if (lane == 0) {
      red[0][0] = lo_x;
      red[1][0] = hi_x;
      red[2][0] = lo_y;
      red[3][0] = hi_y;
    }
  }
  __syncthreads();
  // node window with a one-node margin, clamped to the roi lattice [0, nx] x [0, ny]
  const double fi0 = floor((red[0][0] - r_a - min_x) / res) - 1.0;
  const double fi1 = ceil((red[1][0] + r_a - min_x) / res) + 1.0;
  const double fj0 = floor((red[2][0] - r_a - min_y) / res) - 1.0;
  const double fj1 = ceil((red[3][0] + r_a - min_y) / res) + 1.0;
  if (!(fi0 == fi0 && fi1 == fi1 && fj0 == fj0 && fj1 == fj1)) {
    if (threadIdx.x == 0) *out = 1;
    return;
  }
  const int i0 = static_cast<int>(fmax(fi0, 0.0)), i1 = static_cast<int>(fmin(fi1, double(nx)));
  const int j0 = static_cast<int>(fmax(fj0, 0.0)), j1 = static_cast<int>(fmin(fj1, double(ny)));
  if (i1 < i0 || j1 < j0) return;
  const long long wj = j1 - j0 + 1, cnt = (i1 - i0 + 1) * wj;
  for (long long e = threadIdx.x; e < cnt; e += blockDim.x) {
    const int k = i0 + static_cast<int>(e / wj) - i_org, l = j0 + static_cast<int>(e % wj) - j_org;
    if (k < 0 || k >= ni || l < 0 || l >= nj || P[static_cast<size_t>(k) * nj + l] == 0) {
      *out = 1;
      return;
    }
  }
}

void recursive_update_device(tlg_model* m, const double* x, const double* y, const double* z,
                             size_t mm, bool allow_birth, tlg_update_report* rep,
                             const int* pending_valid) {
  tlg_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  *rep = tlg_update_report{};
  StageTrace tr(ctx);
  // the observation check's flag rides along with the first flag read below
  auto check_valid_now = [&]() {
    if (!pending_valid) return;
    int h = 0;
    TLG_CUDA(cudaMemcpyAsync(&h, pending_valid, sizeof(int), cudaMemcpyDeviceToHost, s));
    TLG_CUDA(cudaStreamSynchronize(s));
    pending_valid = nullptr;
    validate_obs_check(h);
  };

  // ---- births (terrain_model.cpp:150-161) --------------------------------
  if (allow_birth) {
    const tlg_center_params& cp = m->cparams;
    if (!(cp.mesh_resolution > 0.0))
      throw Error(TLG_INVALID_ARGUMENT, "mesh_resolution must be > 0");
    if (cp.accept_count < 1) throw Error(TLG_INVALID_ARGUMENT, "accept_count must be >= 1");
    bool maybe_births = true;
    const double span_x = cp.roi_max_x - cp.roi_min_x, span_y = cp.roi_max_y - cp.roi_min_y;
    if (!m->grid_dirty && m->lat.valid && mm > 0 && span_x >= 0.0 && span_y >= 0.0) {
      const LatticeGrid& L = m->lat;
      int* flag = ctx->ws<int>(S_COUNT, 8);
      TLG_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
      const int rnx = static_cast<int>(std::floor(span_x / cp.mesh_resolution + 1e-9));
      const int rny = static_cast<int>(std::floor(span_y / cp.mesh_resolution + 1e-9));
      k_births_precheck<<<1, 1024, 0, s>>>(x, y, mm, cp.roi_min_x, cp.roi_min_y,
                                           cp.mesh_resolution, cp.accept_radius, rnx, rny,
                                           L.P.p, L.ni, L.nj, L.i_org, L.j_org, flag);
      TLG_LAUNCHED(ctx);
      int hflag = 1, hvalid = 0;
      TLG_CUDA(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
      if (pending_valid)
        TLG_CUDA(cudaMemcpyAsync(&hvalid, pending_valid, sizeof(int), cudaMemcpyDeviceToHost, s));
      TLG_CUDA(cudaStreamSynchronize(s));
      if (pending_valid) {
        pending_valid = nullptr;
        validate_obs_check(hvalid);
      }
      maybe_births = hflag != 0;
    }
    check_valid_now();
    const double *nx = nullptr, *ny = nullptr;
    const size_t nn =
        maybe_births ? supported_nodes_device(ctx, x, y, mm, cp, &nx, &ny) : 0;
    if (nn) {
      std::vector<double> hx(nn), hy(nn);
      TLG_CUDA(cudaMemcpyAsync(hx.data(), nx, nn * 8, cudaMemcpyDeviceToHost, s));
      TLG_CUDA(cudaMemcpyAsync(hy.data(), ny, nn * 8, cudaMemcpyDeviceToHost, s));
      TLG_CUDA(cudaStreamSynchronize(s));
      const size_t first = m->hcx.size();
      std::map<uint32_t, int> old_size;
      for (size_t k = 0; k < nn; ++k) {
        if (m->occupancy.count(mesh_node_key(m, hx[k], hy[k]))) continue;
        const uint32_t b = block_for_tile(m, tile_key(m, hx[k], hy[k]));
        if (!old_size.count(b)) old_size[b] = static_cast<int>(m->members[b].size());
        add_center_host(m, hx[k], hy[k]);
        ++rep->born_centers;
      }
      if (rep->born_centers) {
        upload_new_centres(m, first);
        for (const auto& [b, old] : old_size)
          block_resize(m, b, old, static_cast<int>(m->members[b].size()));
      }
    }
  }
  check_valid_now();
  ensure_grid(m);
  const size_t nc = m->hcx.size();
  const size_t nb = m->members.size();
  if (nc == 0) return;
  tr.mark("births");

  // ---- active set (:163-172) ---------------------------------------------
  const GridView g = grid_view(m);
  uint8_t* active = ctx->ws<uint8_t>(S_ACTIVE, nc);
  uint8_t* bflag = ctx->ws<uint8_t>(S_BLOCKFLAG, nb);
  TLG_CUDA(cudaMemsetAsync(active, 0, nc, s));
  TLG_CUDA(cudaMemsetAsync(bflag, 0, nb, s));
  k_mark_active_w<<<warp_grid(mm, ctx->num_sms), 128, 0, s>>>(g, x, y, mm, m->kc.r2, active);
  TLG_LAUNCHED(ctx);
  k_mark_blocks<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(active, m->d_block_index.p, nc, bflag);
  TLG_LAUNCHED(ctx);
  std::vector<uint8_t> hflag(nb);
  TLG_CUDA(cudaMemcpyAsync(hflag.data(), bflag, nb, cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
  std::vector<uint32_t> ablocks;
  for (uint32_t b = 0; b < nb; ++b)
    if (hflag[b]) ablocks.push_back(b);  // std::set order = ascending ids
  rep->active_blocks = ablocks.size();
  if (ablocks.empty()) return;
  tr.mark("active");
  size_t n_total = 0;
  for (uint32_t b : ablocks) n_total += m->members[b].size();
  // The information form factors H1 = H0 + Mt Mt^T, which couples only
  // blocks whose tiles touch (|dtx|, |dty| <= 1: shared observations lie within
  // the cutoff of both centres, tile side = 2 cutoff). Ordering the merged
  // blocks row by row over the tile grid (the shorter extent fastest) makes
  // H1 block-banded; the band is passed to the factorisation. The Woodbury
  // form keeps the reference's ascending block order.
  const bool info_form = mm > n_total;
  std::vector<std::pair<int64_t, int64_t>> btile;
  if (info_form) btile = spatial_block_order(m, ablocks);

  // ---- merged system (:174-184) ------------------------------------------
  std::vector<uint32_t> merged;
  std::vector<BlockTab> tab(ablocks.size());
  std::vector<int> rowblk, rowloc;
  for (size_t q = 0; q < ablocks.size(); ++q) {
    const uint32_t b = ablocks[q];
    tab[q].pool_off = m->blk_off[b];
    tab[q].ld = m->blk_ld[b];
    tab[q].n = static_cast<int>(m->members[b].size());
    tab[q].off = static_cast<int>(merged.size());
    for (size_t i = 0; i < m->members[b].size(); ++i) {
      merged.push_back(m->members[b][i]);
      rowblk.push_back(static_cast<int>(q));
      rowloc.push_back(static_cast<int>(i));
    }
  }
  const int n = static_cast<int>(merged.size());
  const int nq = static_cast<int>(ablocks.size());
  rep->active_centers = static_cast<uint64_t>(n);
  int maxq = 0;
  for (const auto& t : tab) maxq = std::max(maxq, t.n);
  const int band = btile.empty() ? n : block_band(btile, ablocks, tab);

  // pinned staging for the small host->device tables
  const size_t bytes_merged = n * 4, bytes_tab = nq * sizeof(BlockTab), bytes_rb = n * 4;
  char* stage = static_cast<char*>(ctx->host_stage(bytes_merged + bytes_tab + 2 * bytes_rb + 64));
  std::memcpy(stage, merged.data(), bytes_merged);
  std::memcpy(stage + bytes_merged, tab.data(), bytes_tab);
  std::memcpy(stage + bytes_merged + bytes_tab, rowblk.data(), bytes_rb);
  std::memcpy(stage + bytes_merged + bytes_tab + bytes_rb, rowloc.data(), bytes_rb);
  char* dstage = ctx->ws<char>(S_MERGED, bytes_merged + bytes_tab + 2 * bytes_rb + 64);
  // BlockTab needs 8-byte alignment: place it first in device memory
  BlockTab* d_tab = reinterpret_cast<BlockTab*>(dstage);
  uint32_t* d_merged = reinterpret_cast<uint32_t*>(dstage + bytes_tab);
  int* d_rowblk = reinterpret_cast<int*>(dstage + bytes_tab + bytes_merged);
  int* d_rowloc = reinterpret_cast<int*>(dstage + bytes_tab + bytes_merged + bytes_rb);
  TLG_CUDA(cudaMemcpyAsync(d_tab, stage + bytes_merged, bytes_tab, cudaMemcpyHostToDevice, s));
  TLG_CUDA(cudaMemcpyAsync(d_merged, stage, bytes_merged, cudaMemcpyHostToDevice, s));
  TLG_CUDA(cudaMemcpyAsync(d_rowblk, stage + bytes_merged + bytes_tab, 2 * bytes_rb,
                           cudaMemcpyHostToDevice, s));

  int* rowof = ctx->ws<int>(S_ROWOF, nc);
  TLG_CUDA(cudaMemsetAsync(rowof, 0xff, nc * 4, s));
  k_scatter_rowof<<<(n + 255) / 256, 256, 0, s>>>(d_merged, n, rowof);
  TLG_LAUNCHED(ctx);
  tr.mark("merge");

  // ---- K5: Mt (CSR over observations, cols = merged rows) -----------------
  const Csr c = build_csr(m, x, y, mm, rowof, m->kc.neg_inv_2st2, m->kc.scale, false, nullptr);
  {
    // algorithmic FP64 flops of the formulation about to run:
    // F_W = 2 nnz nbar_q + 2 m^2 kbar + (2/3) m^3 (Cholesky + X) + m^2 n (Y)
    //       + 2 m sum_q n_q^2;
    // F_I = sum_q n_q^3 + 2 m kbar^2 + n b^2 + n^2 b (X) + 2 sum_q (n - off_q) n_q^2
    const double md = static_cast<double>(mm), nd = n, nnz = static_cast<double>(c.nnz);
    const double kbar = mm ? nnz / md : 0.0;
    double s2 = 0.0, s3 = 0.0, st = 0.0;
    for (const auto& tq : tab) {
      const double q = tq.n;
      s2 += q * q;
      s3 += q * q * q;
      st += (nd - tq.off) * q * q;
    }
    rep->flops = info_form ? s3 + 2.0 * md * kbar * kbar + nd * band * double(band) +
                                 nd * nd * band + 2.0 * st
                           : 2.0 * nnz * (nq ? nd / nq : 0.0) + 2.0 * md * md * kbar +
                                 (2.0 / 3.0) * md * md * md + md * md * nd + 2.0 * md * s2;
  }
  double* wm = ctx->ws<double>(S_WORK1, n);
  k_gather_w<<<(n + 255) / 256, 256, 0, s>>>(m->w.p, d_merged, n, wm);
  TLG_LAUNCHED(ctx);
  double* resid = ctx->ws<double>(S_RESID, mm);
  k_residual<<<(unsigned)((mm * 32 + 255) / 256), 256, 0, s>>>(c.rowp, c.col, c.val, z, wm, mm,
                                                                resid);
  TLG_LAUNCHED(ctx);
  tr.mark("csr");

  int* info = ctx->ws<int>(S_FLAGS, 4);
  TLG_CUDA(cudaMemsetAsync(info, 0, 4 * sizeof(int), s));
  double* dw = ctx->ws<double>(S_WORK3, n);
  const int mi = static_cast<int>(mm);
  std::vector<GemmDesc> descs(nq);

  if (!info_form) {
    // ---- (W) one-shot Woodbury ----------------------------------------------
    rep->solver = 1;
    double* Kt = ctx->ws<double>(S_KMAT, static_cast<size_t>(mi) * n);
    TLG_CUDA(cudaMemsetAsync(Kt, 0, sizeof(double) * mi * n, s));
    k_build_Kt<<<mi, 128, 0, s>>>(c.rowp, c.col, c.val, d_rowblk, d_rowloc, d_tab, m->pool.p, mi, Kt);
    TLG_LAUNCHED(ctx);
    double* S = ctx->ws<double>(S_SMAT, static_cast<size_t>(mi) * mi);
    k_build_S<<<mi, 256, 0, s>>>(c.rowp, c.col, c.val, Kt, mi, S);
    TLG_LAUNCHED(ctx);
    tr.mark("K_S");
    symmetrize(ctx, S, mi, mi);
    double* X = ctx->ws<double>(S_XINV, static_cast<size_t>(mi) * mi);
    potrf_lower(ctx, S, mi, mi, info, X, mi);
    int h = 0;
    TLG_CUDA(cudaMemcpyAsync(&h, info, sizeof(int), cudaMemcpyDeviceToHost, s));
    TLG_CUDA(cudaStreamSynchronize(s));
    if (h) {
      rep->rejected = 1;
      return;
    }
    tr.mark("potrf");
    // u = S^-1 r = X^T (X r) ; dw = K u
    double* v = ctx->ws<double>(S_SOLVE, mi);
    gemm(ctx, GemmDesc{mi, 1, mi, X, mi, 0, resid, mi, 0, v, mi, 1.0, 0.0, 2});
    gemm(ctx, GemmDesc{mi, 1, mi, X, mi, 1, v, mi, 0, resid, mi, 1.0, 0.0, 0});
    gemm(ctx, GemmDesc{n, 1, mi, Kt, mi, 1, resid, mi, 0, dw, n, 1.0, 0.0, 0});
    // Y = X K^T ; Hinv1_q = Hinv0_q - Y_q^T Y_q
    double* Y = ctx->ws<double>(S_YMAT, static_cast<size_t>(mi) * n);
    gemm(ctx, GemmDesc{mi, n, mi, X, mi, 0, Kt, mi, 0, Y, mi, 1.0, 0.0, 2});
    tr.mark("trsm");
    for (int q = 0; q < nq; ++q)
      descs[q] = GemmDesc{tab[q].n, tab[q].n, mi, Y + static_cast<size_t>(tab[q].off) * mi, mi, 1,
                          Y + static_cast<size_t>(tab[q].off) * mi, mi, 0,
                          m->pool.p + tab[q].pool_off, tab[q].ld, -1.0, 1.0, 0};
  } else {
    // ---- (I) information form -----------------------------------------------
    rep->solver = 2;
    // the banded Gram keeps a (2 band + 1)-wide window per warp in shared
    // memory; only when that does not fit does the row Gram's n-wide
    // accumulator (n <= 25,600) take over (gram_band)
    require((2.0 * band + 1.0) * 8.0 * kGramWarps <= 200.0 * 1024 ||
                static_cast<size_t>(n) * 8 <= 200 * 1024,
            TLG_RUNTIME_ERROR,
            "information-form update: band of the active blocks too wide for the banded Gram");
    require(static_cast<double>(n) * n * 8.0 * 2.0 <= 64.0 * (1ull << 30), TLG_OUT_OF_MEMORY,
            "information-form update: the dense H and L^-1 workspaces exceed 64 GiB");
    double* H = ctx->ws<double>(S_HMAT, static_cast<size_t>(n) * n);
    TLG_CUDA(cudaMemsetAsync(H, 0, sizeof(double) * n * n, s));
    // H0 = blockdiag(info_inv_q)^-1: all blocks in one launch when they fit
    // in shared memory, else one factorisation per block
    if (maxq <= kBatchInvMax) {
      std::vector<InvJob> jobs(nq);
      for (int q = 0; q < nq; ++q)
        jobs[q] = InvJob{m->pool.p + tab[q].pool_off,
                         H + tab[q].off + static_cast<size_t>(tab[q].off) * n, tab[q].ld, n,
                         tab[q].n, 0};
      batched_spd_inverse(ctx, jobs, info + 1);
    } else {
      for (int q = 0; q < nq; ++q) {
        double* dst = H + tab[q].off + static_cast<size_t>(tab[q].off) * n;
        if (!spd_inverse(ctx, m->pool.p + tab[q].pool_off, tab[q].ld, tab[q].n, dst, n)) {
          rep->rejected = 1;
          return;
        }
      }
    }
    tr.mark("H0");
    // H += Mt Mt^T (lower band; the factorisation reads the lower triangle
    // only) and dw = Mt resid: the lattice element assembly when the centres
    // are mesh nodes, else the row-wise CSR Gram
    TLG_CUDA(cudaMemsetAsync(dw, 0, sizeof(double) * n, s));
    if (m->batch_csr_gram || !lattice_gram_device(m, x, y, resid, mm, rowof, band, H, n, dw)) {
      const TCsr t = transpose_csr(ctx, c, mm, n);
      gram_band(ctx, t, c, n, band, H, n);
      k_row_dot<<<(n + 7) / 8, 256, 0, s>>>(t.rowp, t.obs, t.val, resid, n, dw);
      TLG_LAUNCHED(ctx);
    }
    // X = L^-1 from the factorisation; (H^-1)_qq = X[:,q]^T X[:,q]
    tr.mark("gram");
    double* X = ctx->ws<double>(S_YMAT, static_cast<size_t>(n) * n);
    potrf_lower(ctx, H, n, n, info, X, n, band);
    int h[2] = {0, 0};
    TLG_CUDA(cudaMemcpyAsync(h, info, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    TLG_CUDA(cudaStreamSynchronize(s));
    if (h[0] || h[1]) {
      rep->rejected = 1;
      return;
    }
    tr.mark("potrf");
    double* v = ctx->ws<double>(S_SOLVE, n);
    gemm(ctx, GemmDesc{n, 1, n, X, n, 0, dw, n, 0, v, n, 1.0, 0.0, 2});
    gemm(ctx, GemmDesc{n, 1, n, X, n, 1, v, n, 0, dw, n, 1.0, 0.0, 0});
    tr.mark("solve");
    for (int q = 0; q < nq; ++q) {
      const size_t o = tab[q].off;
      descs[q] = GemmDesc{tab[q].n, tab[q].n, n - tab[q].off, X + o + o * n, n, 1,
                          X + o + o * n, n, 0, m->pool.p + tab[q].pool_off, tab[q].ld, 1.0, 0.0, 0};
    }
  }
  // per-block products, then symmetrise and write back the weights
  GemmDesc* d_descs = reinterpret_cast<GemmDesc*>(ctx->ws<char>(S_BLKTAB, nq * sizeof(GemmDesc)));
  GemmDesc* h_descs = static_cast<GemmDesc*>(ctx->host_stage(nq * sizeof(GemmDesc)));
  std::memcpy(h_descs, descs.data(), nq * sizeof(GemmDesc));
  TLG_CUDA(cudaMemcpyAsync(d_descs, h_descs, nq * sizeof(GemmDesc), cudaMemcpyHostToDevice, s));
  int maxk = 0;
  bool plain = true;
  for (const auto& dq : descs) {
    maxk = std::max(maxk, dq.K);
    plain = plain && dq.uplo == 0;
  }
  tr.mark("descs");
  gemm_grouped(ctx, d_descs, nq, maxq, maxq, plain ? maxk : 0);
  tr.mark("blocks");
  {
    const size_t smem = sizeof(double) * static_cast<size_t>(maxq) * maxq;
    if (smem <= 200 * 1024) {
      if (smem > 48 * 1024)
        TLG_CUDA(cudaFuncSetAttribute(k_symmetrize_blocks,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_symmetrize_blocks<<<nq, 256, smem, s>>>(d_tab, m->pool.p);
    } else {
      k_symmetrize_blocks_global<<<nq, 256, 0, s>>>(d_tab, m->pool.p);
    }
  }
  TLG_LAUNCHED(ctx);
  k_apply_dw<<<(n + 255) / 256, 256, 0, s>>>(m->w.p, d_merged, n, dw);
  TLG_LAUNCHED(ctx);
  sync_weights_to_grid(m);
  TLG_CUDA(cudaStreamSynchronize(s));
}


// ---------------------------------------------------------------------------
// fit_batch_ridge (terrain_model.cpp:269-308): H = lambda I + sum m m^T,
// b = sum m z, w = H^-1 b (Cholesky), info_inv_b = (H_bb)^-1.
__global__ void k_scatter_w(const uint32_t* __restrict__ merged, int n, const double* __restrict__ b,
                            double* __restrict__ w) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) w[merged[r]] = b[r];
}

// terrain_model.cpp:269-308: w = (lambda I + Mt Mt^T)^-1 Mt z and
// info_inv_b = (H_bb)^-1. Rows are merged block by block in the spatial
// order (H is then block-banded: banded Gram, banded 32-wide Cholesky, one
// banded forward/backward solve); the diagonal-block inverses run batched
// before the factorisation overwrites H.
//
// H lives in lower band storage: element (i, j), 0 <= i - j <= kd, at
// H[i + j * ld] with ld = 32 (bwt + 2) (bwt = tile bandwidth) — the dense
// column-major addressing with a short leading dimension (column j's band
// starts at j (ld + 1); n (ld + 1) elements in all), so the tile kernels run
// unchanged; the upper triangles of the diagonal tiles alias only entries
// beyond the band, which nothing reads. When the band covers the matrix,
// ld = n (dense). The split into plan / assemble / solve is the
// point-sharded multi-GPU form: ranks assemble partial systems
// over their point shards, the caller sums them (NCCL all-reduce), every
// rank solves.
// tmp_q (n_q x n_q, ld n_q) <- H_bb at the block's merged rows pos[off..]:
// (max, min) of the two rows in lower band storage, zero beyond the band.
__global__ void k_gather_blocks(const double* __restrict__ H, int ld, int band,
                                const uint32_t* __restrict__ pos, const int* __restrict__ tab,
                                double* __restrict__ tmp) {
  const int q = blockIdx.x;
  const int off = tab[3 * q], nq = tab[3 * q + 1], to = tab[3 * q + 2];
  for (int e = threadIdx.x; e < nq * nq; e += blockDim.x) {
    const int r = e % nq, c = e / nq;
    const int a = static_cast<int>(pos[off + r]), b = static_cast<int>(pos[off + c]);
    const int hi = max(a, b), lo = min(a, b);
    tmp[to + e] = hi - lo <= band ? H[hi + static_cast<size_t>(lo) * ld] : 0.0;
  }
}

struct BatchPlan {
  std::vector<uint32_t> merged;
  std::vector<BlockTab> tab;
  int n = 0, band = 0, ld = 0;
  // node order (lattice models): rows follow the lattice row by row (the
  // shorter extent fastest), blocks are not contiguous; pos lists each
  // block's merged rows in member order (tab[q].off indexes pos)
  bool node_order = false;
  std::vector<uint32_t> pos;
};

// Node-ordered rows for a lattice model: the band of H is then the reach of
// the 2 rho neighbourhood in lattice rows (C5: 2,846 rows instead of 3,424 in
// the block order, ~30 % fewer factorisation flops). Returns false when the
// model is not a lattice.
static bool node_order_plan(tlg_model* m, const std::vector<uint32_t>& blocks, BatchPlan& p) {
  const LatticeGrid& L = m->lat;
  if (!L.valid) return false;
  const size_t nc = m->hcx.size();
  const double res = m->cparams.mesh_resolution;
  const double mnx = m->cparams.roi_min_x, mny = m->cparams.roi_min_y;
  std::vector<int> ni(nc), nj(nc);
  int i0 = INT_MAX, i1 = INT_MIN, j0 = INT_MAX, j1 = INT_MIN;
  for (size_t c = 0; c < nc; ++c) {  // node indices exactly as k_lattice_fill
    ni[c] = static_cast<int>(std::llround((m->hcx[c] - mnx) / res));
    nj[c] = static_cast<int>(std::llround((m->hcy[c] - mny) / res));
    i0 = std::min(i0, ni[c]);
    i1 = std::max(i1, ni[c]);
    j0 = std::min(j0, nj[c]);
    j1 = std::max(j1, nj[c]);
  }
  const long long ei = static_cast<long long>(i1) - i0 + 1, ej = static_cast<long long>(j1) - j0 + 1;
  if (ei * ej > (1ll << 28)) return false;
  const bool j_fast = ej <= ei;
  const long long nf = j_fast ? ej : ei;
  std::vector<int> byslot(static_cast<size_t>(ei * ej), -1);
  for (size_t c = 0; c < nc; ++c) {
    const long long sl = j_fast ? (ni[c] - i0) * ej + (nj[c] - j0) : (nj[c] - j0) * ei + (ni[c] - i0);
    if (byslot[sl] >= 0) return false;  // repeated node (not a lattice after all)
    byslot[sl] = static_cast<int>(c);
  }
  std::vector<uint8_t> inblock(nc, 0);
  for (uint32_t bb : blocks)
    for (uint32_t c : m->members[bb]) inblock[c] = 1;
  std::vector<int> row(nc, -1);
  for (int c : byslot)
    if (c >= 0 && inblock[c]) {
      row[c] = static_cast<int>(p.merged.size());
      p.merged.push_back(static_cast<uint32_t>(c));
    }
  p.tab.resize(blocks.size());
  for (size_t q = 0; q < blocks.size(); ++q) {
    const uint32_t bb = blocks[q];
    p.tab[q].pool_off = m->blk_off[bb];
    p.tab[q].ld = m->blk_ld[bb];
    p.tab[q].n = static_cast<int>(m->members[bb].size());
    p.tab[q].off = static_cast<int>(p.pos.size());
    for (uint32_t c : m->members[bb]) p.pos.push_back(static_cast<uint32_t>(row[c]));
  }
  p.n = static_cast<int>(p.merged.size());
  // entries couple centres within two cutoffs: lattice offsets (di, dj) with
  // (di^2 + dj^2) res^2 <= (2 rho)^2 (with margin); the merged distance of two
  // present nodes is at most their slot distance di nf + dj
  const double reach = 2.0 * m->kernel.cutoff_radius * (1.0 + 1e-9) / res;
  const int R = static_cast<int>(std::ceil(reach)) + 1;
  long long band = 0;
  for (int di = 0; di <= R; ++di)
    for (int dj = -R; dj <= R; ++dj)
      if (static_cast<double>(di) * di + static_cast<double>(dj) * dj <= reach * reach + 1e-9 &&
          (di > 0 || dj > 0))
        band = std::max(band, di * nf + dj);
  p.band = static_cast<int>(std::min<long long>(band, p.n));
  p.node_order = true;
  return true;
}

static BatchPlan batch_plan(tlg_model* m) {
  BatchPlan p;
  std::vector<uint32_t> blocks;
  for (uint32_t bb = 0; bb < m->members.size(); ++bb)
    if (!m->members[bb].empty()) blocks.push_back(bb);
  if (!m->batch_block_order && node_order_plan(m, blocks, p)) {
    constexpr int kTile = 32;
    const long long bwt = (static_cast<long long>(p.band) + kTile - 1) / kTile;
    const long long ldb = (bwt + 2) * kTile;
    if (ldb < p.n) {
      p.ld = static_cast<int>(ldb);
    } else {
      p.ld = p.n;
      p.band = p.n;
    }
    return p;
  }
  const auto btile = spatial_block_order(m, blocks);
  p.tab.resize(blocks.size());
  for (size_t q = 0; q < blocks.size(); ++q) {
    const uint32_t bb = blocks[q];
    p.tab[q].pool_off = m->blk_off[bb];
    p.tab[q].ld = m->blk_ld[bb];
    p.tab[q].n = static_cast<int>(m->members[bb].size());
    p.tab[q].off = static_cast<int>(p.merged.size());
    p.merged.insert(p.merged.end(), m->members[bb].begin(), m->members[bb].end());
  }
  p.n = static_cast<int>(p.merged.size());
  p.band = btile.empty() ? p.n : block_band(btile, blocks, p.tab);
  constexpr int kTile = 32;  // potrf_lower's tile for banded systems (dense.cu NB32)
  const long long bwt = (static_cast<long long>(p.band) + kTile - 1) / kTile;
  const long long ldb = (bwt + 2) * kTile;
  if (ldb < p.n) {
    p.ld = static_cast<int>(ldb);
  } else {
    p.ld = p.n;
    p.band = p.n;
  }
  return p;
}

static size_t batch_elems(const BatchPlan& p) {
  return static_cast<size_t>(p.n) * (static_cast<size_t>(p.ld) + 1);
}

void batch_system_dims(tlg_model* m, size_t* n, size_t* ld, size_t* elems) {
  const BatchPlan p = batch_plan(m);
  *n = static_cast<size_t>(p.n);
  *ld = static_cast<size_t>(p.ld);
  *elems = batch_elems(p);
}

static uint32_t* upload_merged(tlg_ctx* ctx, const BatchPlan& p) {
  cudaStream_t s = ctx->stream;
  uint32_t* hm = static_cast<uint32_t*>(ctx->host_stage(p.n * sizeof(uint32_t)));
  std::memcpy(hm, p.merged.data(), p.n * sizeof(uint32_t));
  uint32_t* d_merged = ctx->ws<uint32_t>(S_MERGED, p.n);
  TLG_CUDA(cudaMemcpyAsync(d_merged, hm, p.n * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
  return d_merged;
}

// H (band storage, ld) <- [lambda I +] Mt Mt^T over this shard, b <- Mt z.
static void batch_assemble(tlg_model* m, const BatchPlan& p, const double* x, const double* y,
                           const double* z, size_t mm, double* H, int ld, double* b,
                           bool add_lambda) {
  tlg_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  const int n = p.n;
  const int nc = static_cast<int>(m->hcx.size());
  TLG_CUDA(cudaMemsetAsync(H, 0, sizeof(double) * batch_elems(p), s));
  TLG_CUDA(cudaMemsetAsync(b, 0, sizeof(double) * n, s));
  if (add_lambda) add_diag(ctx, H, n, ld, m->kernel.lambda);
  if (mm == 0) return;
  const uint32_t* d_merged = upload_merged(ctx, p);
  int* rowof = ctx->ws<int>(S_ROWOF, nc);
  TLG_CUDA(cudaMemsetAsync(rowof, 0xff, nc * 4, s));
  k_scatter_rowof<<<(n + 255) / 256, 256, 0, s>>>(d_merged, n, rowof);
  TLG_LAUNCHED(ctx);
  if (!m->batch_csr_gram && lattice_gram_device(m, x, y, z, mm, rowof, p.band, H, ld, b)) return;
  const Csr c = build_csr(m, x, y, mm, rowof, m->kc.neg_inv_2st2, m->kc.scale, false, nullptr);
  const TCsr t = transpose_csr(ctx, c, mm, n);
  gram_band(ctx, t, c, n, p.band, H, ld, /*lower_only=*/true);
  k_row_dot<<<(n + 7) / 8, 256, 0, s>>>(t.rowp, t.obs, t.val, z, n, b);
  TLG_LAUNCHED(ctx);
}

// info_inv_b = (H_bb)^-1 (:298-306) from H before it is factored, then the
// banded Cholesky solve; w scattered back to centre order.
static void batch_solve(tlg_model* m, const BatchPlan& p, double* H, int ld, double* b) {
  tlg_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  const int n = p.n;
  StageTrace tr(ctx);
  const uint32_t* d_merged = upload_merged(ctx, p);
  int* info = ctx->ws<int>(S_FLAGS, 4);
  TLG_CUDA(cudaMemsetAsync(info, 0, 4 * sizeof(int), s));
  int maxq = 0;
  for (const auto& tq : p.tab) maxq = std::max(maxq, tq.n);
  if (p.node_order) {
    // blocks are scattered over the node-ordered rows: gather each H_bb
    // (entries beyond the band are structurally zero) into a dense n_q^2
    // buffer, then invert them batched
    std::vector<size_t> toff(p.tab.size() + 1, 0);
    for (size_t q = 0; q < p.tab.size(); ++q)
      toff[q + 1] = toff[q] + static_cast<size_t>(p.tab[q].n) * p.tab[q].n;
    const size_t npos = p.pos.size();
    uint32_t* hp = static_cast<uint32_t*>(ctx->host_stage(npos * 4 + (p.tab.size() + 1) * 16));
    std::memcpy(hp, p.pos.data(), npos * 4);
    int* htab = reinterpret_cast<int*>(hp + npos);
    for (size_t q = 0; q < p.tab.size(); ++q) {
      htab[3 * q] = p.tab[q].off;
      htab[3 * q + 1] = p.tab[q].n;
      htab[3 * q + 2] = static_cast<int>(toff[q]);
    }
    uint32_t* dpos = ctx->ws<uint32_t>(S_TKEYS, npos + 3 * p.tab.size() + 4);
    int* dtab = reinterpret_cast<int*>(dpos + npos);
    TLG_CUDA(cudaMemcpyAsync(dpos, hp, npos * 4 + 3 * p.tab.size() * 4, cudaMemcpyHostToDevice, s));
    double* tmp = ctx->ws<double>(S_SOLVE, toff.back());
    k_gather_blocks<<<static_cast<unsigned>(p.tab.size()), 256, 0, s>>>(H, ld, p.band, dpos, dtab,
                                                                        tmp);
    TLG_LAUNCHED(ctx);
    if (maxq <= kBatchInvMax) {
      std::vector<InvJob> jobs(p.tab.size());
      for (size_t q = 0; q < p.tab.size(); ++q)
        jobs[q] = InvJob{tmp + toff[q], m->pool.p + p.tab[q].pool_off, p.tab[q].n, p.tab[q].ld,
                         p.tab[q].n, 0};
      batched_spd_inverse(ctx, jobs, info + 1);
    } else {
      for (size_t q = 0; q < p.tab.size(); ++q)
        if (!spd_inverse(ctx, tmp + toff[q], p.tab[q].n, p.tab[q].n, m->pool.p + p.tab[q].pool_off,
                         p.tab[q].ld))
          throw Error(TLG_RUNTIME_ERROR, "ridge solve failed (block factorisation)");
    }
  } else if (maxq <= kBatchInvMax) {
    std::vector<InvJob> jobs(p.tab.size());
    for (size_t q = 0; q < p.tab.size(); ++q)
      jobs[q] = InvJob{H + p.tab[q].off + static_cast<size_t>(p.tab[q].off) * ld,
                       m->pool.p + p.tab[q].pool_off, ld, p.tab[q].ld, p.tab[q].n, 0};
    batched_spd_inverse(ctx, jobs, info + 1);
  } else {
    require(ld == n, TLG_RUNTIME_ERROR, "batch ridge: blocks too large for band storage");
    for (size_t q = 0; q < p.tab.size(); ++q)
      if (!spd_inverse(ctx, H + p.tab[q].off + static_cast<size_t>(p.tab[q].off) * ld, ld,
                       p.tab[q].n, m->pool.p + p.tab[q].pool_off, p.tab[q].ld))
        throw Error(TLG_RUNTIME_ERROR, "ridge solve failed (block factorisation)");
  }
  tr.mark("block_inv");
  potrf_lower(ctx, H, n, ld, info, nullptr, 0, p.band);
  tr.mark("potrf");
  double* mnx = ctx->ws<double>(S_PARTIALS, 2);
  k_diag_minmax<<<1, 256, 0, s>>>(H, n, ld, mnx);
  TLG_LAUNCHED(ctx);
  band_solve(ctx, H, n, ld, p.band, b);
  tr.mark("band_solve");
  int h[2] = {0, 0};
  double cond[2];
  TLG_CUDA(cudaMemcpyAsync(h, info, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaMemcpyAsync(cond, mnx, sizeof(cond), cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
  if (h[1]) throw Error(TLG_RUNTIME_ERROR, "ridge solve failed (block factorisation)");
  if (h[0])
    throw Error(TLG_RUNTIME_ERROR, "ridge solve failed; condition estimate " +
                                       std::to_string(cond[0] / std::max(cond[1], 1e-300)));
  k_scatter_w<<<(n + 255) / 256, 256, 0, s>>>(d_merged, n, b, m->w.p);
  TLG_LAUNCHED(ctx);
  sync_weights_to_grid(m);
  TLG_CUDA(cudaStreamSynchronize(s));
}

void batch_fit_device(tlg_model* m, const double* x, const double* y, const double* z,
                      size_t mm) {
  ensure_grid(m);
  if (m->hcx.empty()) return;
  const BatchPlan p = batch_plan(m);
  require(batch_elems(p) * 8 <= (size_t{64} << 30), TLG_OUT_OF_MEMORY,
          "batch ridge fit: the banded system exceeds 64 GiB of device memory");
  double* H = m->ctx->ws<double>(S_HMAT, batch_elems(p));
  double* b = m->ctx->ws<double>(S_WORK3, p.n);
  batch_assemble(m, p, x, y, z, mm, H, p.ld, b, true);
  batch_solve(m, p, H, p.ld, b);
}

void batch_assemble_device(tlg_model* m, const double* x, const double* y, const double* z,
                           size_t mm, double* H, size_t ld, double* b, bool add_lambda) {
  ensure_grid(m);
  if (m->hcx.empty()) return;
  const BatchPlan p = batch_plan(m);
  require(ld == static_cast<size_t>(p.ld), TLG_INVALID_ARGUMENT,
          "batch ridge: ld differs from tlg_batch_ridge_system");
  batch_assemble(m, p, x, y, z, mm, H, p.ld, b, add_lambda);
  TLG_CUDA(cudaStreamSynchronize(m->ctx->stream));
}

void batch_solve_device(tlg_model* m, double* H, size_t ld, double* b) {
  ensure_grid(m);
  if (m->hcx.empty()) return;
  const BatchPlan p = batch_plan(m);
  require(ld == static_cast<size_t>(p.ld), TLG_INVALID_ARGUMENT,
          "batch ridge: ld differs from tlg_batch_ridge_system");
  batch_solve(m, p, H, p.ld, b);
}

// ---- structural sparsity of the batch system (point-sharded reduction) ----
// Column j of the band storage holds rows i in [j, j + ld) at H[i + j ld];
// entry (i, j) can be nonzero only when one observation lies within the
// cutoff of both centres, i.e. |c_i - c_j| <= 2 cutoff (the diagonal always).
// Counting pass then a fill pass in column order -> deterministic positions.
__global__ void k_bpat_count(const uint32_t* __restrict__ merged, const double* __restrict__ cx,
                             const double* __restrict__ cy, int n, int ld, double r2,
                             uint32_t* __restrict__ cnt) {
  const int j = blockIdx.x;
  const double xj = cx[merged[j]], yj = cy[merged[j]];
  const int i1 = min(n, j + ld);
  uint32_t c = 0;
  for (int i = j + threadIdx.x; i < i1; i += blockDim.x) {
    const double dx = cx[merged[i]] - xj, dy = cy[merged[i]] - yj;
    c += (i == j || dx * dx + dy * dy <= r2) ? 1u : 0u;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ uint32_t sh[32];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    cnt[j] = t;
  }
}

__global__ void k_bpat_fill(const uint32_t* __restrict__ merged, const double* __restrict__ cx,
                            const double* __restrict__ cy, int n, int ld, double r2,
                            const uint32_t* __restrict__ off, uint64_t* __restrict__ pos) {
  const int j = blockIdx.x;
  if (threadIdx.x != 0) return;  // one thread per column keeps row order (cheap: ld tests)
  const double xj = cx[merged[j]], yj = cy[merged[j]];
  const int i1 = min(n, j + ld);
  uint32_t k = off[j];
  for (int i = j; i < i1; ++i) {
    const double dx = cx[merged[i]] - xj, dy = cy[merged[i]] - yj;
    if (i == j || dx * dx + dy * dy <= r2) pos[k++] = static_cast<uint64_t>(i) + static_cast<uint64_t>(j) * ld;
  }
}

__global__ void k_bpat_gather(const uint64_t* __restrict__ pos, size_t nnz, const double* __restrict__ H,
                              double* __restrict__ packed) {
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < nnz; k += (size_t)gridDim.x * blockDim.x)
    packed[k] = H[pos[k]];
}

__global__ void k_bpat_scatter(const uint64_t* __restrict__ pos, size_t nnz, const double* __restrict__ packed,
                               double* __restrict__ H) {
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < nnz; k += (size_t)gridDim.x * blockDim.x)
    H[pos[k]] = packed[k];
}

static size_t batch_pattern(tlg_model* m, const BatchPlan& p) {
  if (m->bpat_for == m->hcx.size() && m->bpat_nnz) return m->bpat_nnz;
  tlg_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  const int n = p.n;
  const uint32_t* d_merged = upload_merged(ctx, p);
  const double rr = 2.0 * m->kernel.cutoff_radius;
  const double r2 = rr * rr * (1.0 + 1e-9);  // a superset of the true pattern
  uint32_t* cnt = ctx->ws<uint32_t>(S_TROWP, n + 1);
  k_bpat_count<<<n, 256, 0, s>>>(d_merged, m->cx.p, m->cy.p, n, p.ld, r2, cnt);
  TLG_LAUNCHED(ctx);
  std::vector<uint32_t> h(n + 1, 0);
  TLG_CUDA(cudaMemcpyAsync(h.data(), cnt, n * 4, cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
  size_t total = 0;
  for (int j = 0; j < n; ++j) {
    const uint32_t c = h[j];
    h[j] = static_cast<uint32_t>(total);
    total += c;
  }
  require(total < (size_t{1} << 32), TLG_RUNTIME_ERROR, "batch pattern too large");
  TLG_CUDA(cudaMemcpyAsync(cnt, h.data(), n * 4, cudaMemcpyHostToDevice, s));
  m->bpat.ensure(total + 1);
  k_bpat_fill<<<n, 32, 0, s>>>(d_merged, m->cx.p, m->cy.p, n, p.ld, r2, cnt, m->bpat.p);
  TLG_LAUNCHED(ctx);
  TLG_CUDA(cudaStreamSynchronize(s));
  m->bpat_nnz = total;
  m->bpat_for = m->hcx.size();
  return total;
}

size_t batch_pattern_device(tlg_model* m) {
  ensure_grid(m);
  if (m->hcx.empty()) return 0;
  return batch_pattern(m, batch_plan(m));
}

void batch_pack_device(tlg_model* m, const double* H, double* packed) {
  const size_t nnz = batch_pattern_device(m);
  if (!nnz) return;
  const unsigned b = static_cast<unsigned>(std::min<size_t>((nnz + 255) / 256, 8ull * m->ctx->num_sms));
  k_bpat_gather<<<b, 256, 0, m->ctx->stream>>>(m->bpat.p, nnz, H, packed);
  TLG_LAUNCHED(m->ctx);
  TLG_CUDA(cudaStreamSynchronize(m->ctx->stream));
}

void batch_unpack_device(tlg_model* m, const double* packed, double* H) {
  const size_t nnz = batch_pattern_device(m);
  const BatchPlan p = batch_plan(m);
  TLG_CUDA(cudaMemsetAsync(H, 0, sizeof(double) * batch_elems(p), m->ctx->stream));
  if (!nnz) return;
  const unsigned b = static_cast<unsigned>(std::min<size_t>((nnz + 255) / 256, 8ull * m->ctx->num_sms));
  k_bpat_scatter<<<b, 256, 0, m->ctx->stream>>>(m->bpat.p, nnz, packed, H);
  TLG_LAUNCHED(m->ctx);
  TLG_CUDA(cudaStreamSynchronize(m->ctx->stream));
}

}  // namespace tlg
