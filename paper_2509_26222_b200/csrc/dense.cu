// Dense FP64 kernels for the kernel-matrix update: a DMMA (mma.sync
// m8n8k4 f64, the sm_100a FP64 tensor path — tcgen05 has no f64 kind) GEMM
// with 64x64 CTA tiles; a tile Cholesky in ONE cooperative launch (per 64-wide
// step: the diagonal tile is factored and inverted in shared memory by one
// CTA, panel tiles become GEMMs with that inverse, trailing tiles are DMMA
// GEMMs, grid barriers between the phases); and a one-launch tile TRSM where
// each CTA walks the tile rows of its 64-column slab with GEMMs only.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "dense.cuh"
#include "dense_tile.cuh"

namespace cg = cooperative_groups;

#ifndef TLG_PHASE
#define TLG_PHASE(k)
#endif
#ifndef TLG_COOP_MARK
#define TLG_COOP_MARK(k, step)
#endif

namespace tlg {

constexpr int TM = 64, TN = 64, TK = 16, SP = 68;  // smem pitch (doubles): conflict-free frags

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// One right-hand side (N == 1): 64 rows of y = alpha op(A) b + beta y with
// plain FMAs (coalesced along the contiguous dimension of A). All reads of b
// finish before y is written, so b may alias y (in-place triangular steps).
__device__ __forceinline__ void gemv_tile(const GemmDesc& d, int m0, int K) {
  __shared__ double red[128];
  const int t = threadIdx.x;
  const int mb = min(TM, d.M - m0);
  auto bval = [&](int k) { return d.tb ? d.B[(size_t)k * d.ldb] : d.B[k]; };
  if (!d.ta) {
    // two threads per row (k even / odd), eight independent partial sums
    // each: eight loads in flight per thread instead of one dependent chain
    const int i = t & 63, h = t >> 6;
    double s[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (i < mb) {
      const double* a = d.A + m0 + i;
      int k = h;
      for (; k + 14 < K; k += 16) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          s[u] = fma(a[(size_t)(k + 2 * u) * d.lda], bval(k + 2 * u), s[u]);
      }
      for (; k < K; k += 2) s[0] = fma(a[(size_t)k * d.lda], bval(k), s[0]);
    }
    red[t] = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
  } else {
    // a warp per row (lanes over k, coalesced), four rows in flight per warp
    const int lane = t & 31, w = t >> 5;
    for (int i0 = w; i0 < mb; i0 += 16) {
      double sr[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + 4 * u;
        if (i < mb) {
          const double* a = d.A + (size_t)(m0 + i) * d.lda;
          for (int k = lane; k < K; k += 32) sr[u] = fma(a[k], bval(k), sr[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sr[u] += __shfl_xor_sync(0xffffffffu, sr[u], o);
        if (lane == 0 && i0 + 4 * u < mb) red[i0 + 4 * u] = sr[u];
      }
    }
  }
  __syncthreads();
  if (t < mb) {
    const double v = d.alpha * (d.ta ? red[t] : red[t] + red[t + 64]);
    double* p = d.C + m0 + t;
    *p = (d.beta == 0.0) ? v : fma(d.beta, *p, v);
  }
  __syncthreads();
}

__device__ __forceinline__ void gemm_tile(const GemmDesc& d, int tile_m, int tile_n) {
  const int m0 = tile_m * TM, n0 = tile_n * TN;
  if (m0 >= d.M || n0 >= d.N) return;
  if (d.uplo == 1 && m0 + TM <= n0) return;  // strictly above the diagonal
  // uplo 2: A lower triangular (not transposed) -> its columns >= m0 + TM are 0
  const int K = (d.uplo == 2) ? min(d.K, m0 + TM) : d.K;
  if (d.N == 1) {
    gemv_tile(d, m0, K);
    return;
  }
  __shared__ double As[TK][SP];
  __shared__ double Bs[TK][SP];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int wm = (w & 1) * 32, wn = (w >> 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // Global -> register prefetch of the next K chunk overlaps the DMMA work of
  // the current one (the tiles are small; latency, not bandwidth, dominates).
  double pa[8], pb[8];
  auto fetch = [&](int k0) {
    if (!d.ta) {
      const int i = t & 63;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int k = (t >> 6) + 2 * s, gi = m0 + i, gk = k0 + k;
        pa[s] = (gi < d.M && gk < K) ? d.A[gi + (size_t)gk * d.lda] : 0.0;
      }
    } else {
      const int k = t & 15;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int i = (t >> 4) + 8 * s, gi = m0 + i, gk = k0 + k;
        pa[s] = (gi < d.M && gk < K) ? d.A[gk + (size_t)gi * d.lda] : 0.0;
      }
    }
    if (!d.tb) {
      const int k = t & 15;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int j = (t >> 4) + 8 * s, gj = n0 + j, gk = k0 + k;
        pb[s] = (gj < d.N && gk < K) ? d.B[gk + (size_t)gj * d.ldb] : 0.0;
      }
    } else {
      const int j = t & 63;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int k = (t >> 6) + 2 * s, gj = n0 + j, gk = k0 + k;
        pb[s] = (gj < d.N && gk < K) ? d.B[gj + (size_t)gk * d.ldb] : 0.0;
      }
    }
  };
  if (K > 0) fetch(0);
  for (int k0 = 0; k0 < K; k0 += TK) {
    // stage chunk: op(A)(m0 + i, k0 + k) -> As[k][i], op(B)(k0 + k, n0 + j) -> Bs[k][j]
    if (!d.ta) {
#pragma unroll
      for (int s = 0; s < 8; ++s) As[(t >> 6) + 2 * s][t & 63] = pa[s];
    } else {
#pragma unroll
      for (int s = 0; s < 8; ++s) As[t & 15][(t >> 4) + 8 * s] = pa[s];
    }
    if (!d.tb) {
#pragma unroll
      for (int s = 0; s < 8; ++s) Bs[t & 15][(t >> 4) + 8 * s] = pb[s];
    } else {
#pragma unroll
      for (int s = 0; s < 8; ++s) Bs[(t >> 6) + 2 * s][t & 63] = pb[s];
    }
    __syncthreads();
    if (k0 + TK < K) fetch(k0 + TK);
#pragma unroll
    for (int kk = 0; kk < TK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk + (lane & 3)][wm + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk + (lane & 3)][wn + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = m0 + wm + i * 8 + (lane >> 2);
        const int c = n0 + wn + j * 8 + 2 * (lane & 3) + h;
        if (r < d.M && c < d.N) {
          double* p = d.C + r + (size_t)c * d.ldc;
          const double v = d.alpha * acc[i][j][h];
          *p = (d.beta == 0.0) ? v : fma(d.beta, *p, v);
        }
      }
}

__global__ void __launch_bounds__(128) k_gemm(GemmDesc d) { gemm_tile(d, blockIdx.x, blockIdx.y); }

__global__ void __launch_bounds__(128) k_gemm_grouped(const GemmDesc* __restrict__ ds) {
  const GemmDesc d = ds[blockIdx.z];
  gemm_tile(d, blockIdx.x, blockIdx.y);
}

// One right-hand side with long K and few row tiles (the update's
// y = X v with X = L^-1, n = 4096: 64 row tiles): split K over CTAs so every
// SM streams A, partial y per slice, then an order-fixed sum.
__global__ void __launch_bounds__(128) k_gemv_splitk(GemmDesc d, int kslice, double* __restrict__ part) {
  const int m0 = blockIdx.x * TM, s2 = blockIdx.y;
  const int k_hi = (d.uplo == 2) ? min(d.K, m0 + TM) : d.K;
  const int k_lo = s2 * kslice;
  double* P = part + (size_t)s2 * d.M;
  if (k_lo >= k_hi) {
    if (threadIdx.x < TM && m0 + threadIdx.x < d.M) P[m0 + threadIdx.x] = 0.0;
    return;
  }
  GemmDesc e = d;
  e.A += e.ta ? k_lo : (size_t)k_lo * e.lda;
  e.B += e.tb ? (size_t)k_lo * e.ldb : k_lo;
  e.K = min(kslice, k_hi - k_lo);
  e.C = P;
  e.ldc = d.M;
  e.alpha = 1.0;
  e.beta = 0.0;
  e.uplo = 0;
  gemv_tile(e, m0, e.K);
}

__global__ void k_gemv_reduce(GemmDesc d, int splits, const double* __restrict__ part) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= d.M) return;
  double v = 0.0;
  for (int s2 = 0; s2 < splits; ++s2) v += part[(size_t)s2 * d.M + r];
  v *= d.alpha;
  double* p = d.C + r;
  *p = (d.beta == 0.0) ? v : fma(d.beta, *p, v);
}

void gemm(tlg_ctx* ctx, const GemmDesc& d) {
  if (d.M <= 0 || d.N <= 0) return;
  const int tm = (d.M + TM - 1) / TM;
  if (d.N == 1 && d.K >= 1024 && tm < 2 * ctx->num_sms) {
    const int splits = std::max(1, std::min((4 * ctx->num_sms + tm - 1) / tm, d.K / 256));
    const int kslice = (d.K + splits - 1) / splits;
    // the partial rows live in the output's workspace-free slot (b may alias C)
    double* part = ctx->ws<double>(S_GEMVPART, static_cast<size_t>(splits) * d.M);
    k_gemv_splitk<<<dim3(tm, splits), 128, 0, ctx->stream>>>(d, kslice, part);
    TLG_LAUNCHED(ctx);
    k_gemv_reduce<<<(d.M + 255) / 256, 256, 0, ctx->stream>>>(d, splits, part);
    TLG_LAUNCHED(ctx);
    return;
  }
  dim3 grid((d.M + TM - 1) / TM, (d.N + TN - 1) / TN);
  k_gemm<<<grid, 128, 0, ctx->stream>>>(d);
  TLG_LAUNCHED(ctx);
}

// Split-K grouped GEMM: CTA (tm, tn, q * S + s) runs descriptor q over its
// s-th K slice into a private partial tile; k_gemm_splitk_reduce sums the S
// slices in order (deterministic) and applies alpha / beta. For few, small
// outputs with long K (the update's per-block X_q^T X_q products: ~50 blocks
// of 84 x 84, K up to n) the plain grouped GEMM leaves most SMs idle.
__global__ void __launch_bounds__(128) k_gemm_grouped_splitk(const GemmDesc* __restrict__ ds, int splits,
                                                             int kslice, double* __restrict__ part,
                                                             int ldp, size_t pstride) {
  const int q = blockIdx.z / splits, sidx = blockIdx.z % splits;
  GemmDesc d = ds[q];
  const int k_lo = sidx * kslice;
  if (k_lo >= d.K || d.uplo != 0) {
    if (d.uplo == 0) {  // an empty slice still owns its partial tile
      const int m0 = blockIdx.x * TM, n0 = blockIdx.y * TN;
      double* P = part + blockIdx.z * pstride;
      for (int e = threadIdx.x; e < TM * TN; e += 128) {
        const int r = m0 + (e & 63), c = n0 + (e >> 6);
        if (r < d.M && c < d.N) P[r + (size_t)c * ldp] = 0.0;
      }
    }
    return;
  }
  d.A += d.ta ? k_lo : (size_t)k_lo * d.lda;
  d.B += d.tb ? (size_t)k_lo * d.ldb : k_lo;
  d.K = min(kslice, d.K - k_lo);
  d.C = part + blockIdx.z * pstride;
  d.ldc = ldp;
  d.alpha = 1.0;
  d.beta = 0.0;
  gemm_tile(d, blockIdx.x, blockIdx.y);
}

__global__ void k_gemm_splitk_reduce(const GemmDesc* __restrict__ ds, int splits,
                                     const double* __restrict__ part, int ldp, size_t pstride,
                                     int max_m, int max_n) {
  const int q = blockIdx.y;
  const GemmDesc d = ds[q];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < max_m * max_n; e += gridDim.x * blockDim.x) {
    const int r = e % max_m, c = e / max_m;
    if (r >= d.M || c >= d.N) continue;
    double v = 0.0;
    for (int s2 = 0; s2 < splits; ++s2) v += part[(q * splits + s2) * pstride + r + (size_t)c * ldp];
    double* p = d.C + r + (size_t)c * d.ldc;
    v *= d.alpha;
    *p = (d.beta == 0.0) ? v : fma(d.beta, *p, v);
  }
}

void gemm_grouped(tlg_ctx* ctx, const GemmDesc* d_descs, int count, int max_m, int max_n, int max_k) {
  if (count <= 0 || max_m <= 0 || max_n <= 0) return;
  const int tm = (max_m + TM - 1) / TM, tn = (max_n + TN - 1) / TN;
  const long long tiles = static_cast<long long>(tm) * tn * count;
  // slices of >= 256 along K until ~4 CTAs per SM are busy
  int splits = 1;
  if (max_k > 512) {
    const long long want = (4ll * ctx->num_sms + tiles - 1) / tiles;
    splits = static_cast<int>(std::max(1ll, std::min<long long>(want, max_k / 256)));
  }
  if (splits == 1) {
    dim3 grid(tm, tn, count);
    k_gemm_grouped<<<grid, 128, 0, ctx->stream>>>(d_descs);
    TLG_LAUNCHED(ctx);
    return;
  }
  const int kslice = ((max_k + splits - 1) / splits + TK - 1) / TK * TK;
  const int ldp = tm * TM;
  const size_t pstride = static_cast<size_t>(ldp) * tn * TN;
  // own slot, sized for ~4 CTAs per SM of partial tiles plus one per tile
  // (tiles x splits never exceeds that): it does not regrow when the block
  // count shifts between scans (a regrowth is a cudaFree + cudaMalloc pair,
  // measured at up to tens of ms mid-stream)
  const size_t cap = static_cast<size_t>(4ll * ctx->num_sms + tiles) * TM * TN;
  double* part = ctx->ws<double>(S_GGPART, std::max(cap, pstride * count * splits));
  dim3 grid(tm, tn, count * splits);
  k_gemm_grouped_splitk<<<grid, 128, 0, ctx->stream>>>(d_descs, splits, kslice, part, ldp, pstride);
  TLG_LAUNCHED(ctx);
  dim3 rgrid(static_cast<unsigned>(std::min(64, (max_m * max_n + 255) / 256)), count);
  k_gemm_splitk_reduce<<<rgrid, 256, 0, ctx->stream>>>(d_descs, splits, part, ldp, pstride, max_m, max_n);
  TLG_LAUNCHED(ctx);
}


// ---------------------------------------------------------------------------
// Tile factorisation. NB = 64-wide tiles; every tile step is one CTA of 128
// threads running gemm_tile (DMMA) or the diagonal-tile routine below.
constexpr int NB = 64;

// Diagonal tile L L^T = A (64 x 64, 128 threads) and X = L^-1 with one-panel
// lookahead. Panels are 4 columns wide. In phase J warp 0 brings panel J+1
// up to date (rank-4 update of its 4 columns and of X rows j+4..j+7) and
// factors it, while warps 1-3 apply the panel-J rank-4 update to the rest of
// the trailing matrix and of X. One barrier per phase; the critical path is
// warp 0's small panel chain instead of panel + whole trailing update.
// Shared memory: A and X column-major with odd pitch kLaP (lanes may walk rows
// or columns without bank conflicts); the published panel is kept twice —
// PLr[q][64] (lane = row reads) and PLc[64][4] (broadcast reads) — and so are
// the final X rows, PXr[q][64] and PXc[64][4]; each is double-buffered by phase.
constexpr int kLaP = 65;
constexpr int kLaPanel = 4 * 64;  // doubles per published panel copy
constexpr int kDiagSmemDoubles = 2 * 64 * kLaP + 2 + 8 * kLaPanel;

struct LaBuf {
  const double* PLr;
  const double* PLc;
  const double* PXr;
  const double* PXc;
};

__device__ __forceinline__ void la_factor4(const double (&D)[4][4], double (&L)[4][4],
                                           double (&Li)[4][4], bool& bad) {
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    double d = D[p][p];
#pragma unroll
    for (int k = 0; k < p; ++k) d = fma(-L[p][k], L[p][k], d);
    bad |= !(d > 0.0) || !isfinite(d);
    const double iv = rsqrt(d);
    L[p][p] = d * iv;
    Li[p][p] = iv;
#pragma unroll
    for (int r = p + 1; r < 4; ++r) {
      double s = D[r][p];
#pragma unroll
      for (int k = 0; k < p; ++k) s = fma(-L[r][k], L[p][k], s);
      L[r][p] = s * iv;
    }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int r = c + 1; r < 4; ++r) {
      double s = 0.0;
#pragma unroll
      for (int k = c; k < r; ++k) s = fma(L[r][k], Li[k][c], s);
      Li[r][c] = -Li[r][r] * s;
    }
}

// Warp 0: panel jn (columns jn..jn+3) — update with the previous panel (when
// jn > 0), factor, and publish L rows and final X rows into `out`.
__device__ __forceinline__ void la_panel(double* __restrict__ a, double* __restrict__ x,
                                         const LaBuf& o, double* __restrict__ PLr,
                                         double* __restrict__ PLc, double* __restrict__ PXr,
                                         double* __restrict__ PXc, int jn, bool& bad) {
  const int l = threadIdx.x & 31;
  double ar[2][4], xr[2][4];
  double lp[4][4];  // L rows jn..jn+3 of the previous panel (broadcast)
  if (jn > 0) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const double2 u = *reinterpret_cast<const double2*>(o.PLc + (jn + p) * 4);
      const double2 v = *reinterpret_cast<const double2*>(o.PLc + (jn + p) * 4 + 2);
      lp[p][0] = u.x;
      lp[p][1] = u.y;
      lp[p][2] = v.x;
      lp[p][3] = v.y;
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = jn + l + 32 * h;
    if (r < 64) {
#pragma unroll
      for (int p = 0; p < 4; ++p) ar[h][p] = a[(jn + p) * kLaP + r];
      if (jn > 0) {
        double lr[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) lr[q] = o.PLr[q * 64 + r];
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) ar[h][p] = fma(-lr[q], lp[p][q], ar[h][p]);
        if (r < jn + 4)
#pragma unroll
          for (int p = 0; p < 4; ++p) a[(jn + p) * kLaP + r] = ar[h][p];
      }
    }
    const int c = l + 32 * h;
    if (c < jn) {
#pragma unroll
      for (int p = 0; p < 4; ++p) xr[h][p] = x[c * kLaP + jn + p];
      double xo[4];  // X_fin rows of the previous panel: nonzero in columns < jn
#pragma unroll
      for (int q = 0; q < 4; ++q) xo[q] = o.PXr[q * 64 + c];
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) xr[h][p] = fma(-lp[p][q], xo[q], xr[h][p]);
    }
  }
  TLG_PHASE(1);
  __syncwarp();
  double D[4][4], L[4][4], Li[4][4];
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q <= p; ++q) D[p][q] = a[(jn + q) * kLaP + jn + p];
  TLG_PHASE(2);
  la_factor4(D, L, Li, bad);
  TLG_PHASE(3);
  // L rows: r in the diagonal block take L; rows below: a_r Li^T
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = jn + l + 32 * h;
    if (r < 64) {
      double v[4];
      if (r >= jn + 4) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double s = 0.0;
#pragma unroll
          for (int p = 0; p <= q; ++p) s = fma(ar[h][p], Li[q][p], s);
          v[q] = s;
        }
      } else {
        const int pr = r - jn;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double s = 0.0;
#pragma unroll
          for (int p = 0; p < 4; ++p)
            if (p == pr) s = q <= p ? L[p][q] : 0.0;
          v[q] = s;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[(jn + q) * kLaP + r] = v[q];
        PLr[q * 64 + r] = v[q];
      }
      *reinterpret_cast<double2*>(PLc + r * 4) = make_double2(v[0], v[1]);
      *reinterpret_cast<double2*>(PLc + r * 4 + 2) = make_double2(v[2], v[3]);
    }
  }
  TLG_PHASE(4);
  // final X rows jn..jn+3: Li X(rows); columns < jn from the update, jn.. = I
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = l + 32 * h;
    double xi[4];
    if (c < jn) {
#pragma unroll
      for (int p = 0; p < 4; ++p) xi[p] = xr[h][p];
    } else {
#pragma unroll
      for (int p = 0; p < 4; ++p) xi[p] = (c == jn + p) ? 1.0 : 0.0;
    }
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double s = 0.0;
#pragma unroll
      for (int p = 0; p <= q; ++p) s = fma(Li[q][p], xi[p], s);
      v[q] = s;
      if (c <= jn + 3) x[c * kLaP + jn + q] = s;
      PXr[q * 64 + c] = s;
    }
    *reinterpret_cast<double2*>(PXc + c * 4) = make_double2(v[0], v[1]);
    *reinterpret_cast<double2*>(PXc + c * 4 + 2) = make_double2(v[2], v[3]);
  }
}

__device__ void tile_potrf_inv_la(double* __restrict__ A, int lda, int kb,
                                  double* __restrict__ linv, int* __restrict__ info,
                                  double* sh) {
  const int t = threadIdx.x;
  double* a = sh;                  // A, column-major [64][kLaP]
  double* x = sh + 64 * kLaP;      // X, column-major [64][kLaP]
  double* pb = sh + 2 * 64 * kLaP + 2;  // 16-byte aligned panel buffers
  auto buf = [&](int which, int parity) { return pb + (which * 2 + parity) * kLaPanel; };
  for (int e = t; e < 64 * 64; e += 128) {
    const int r = e & 63, c = e >> 6;
    a[c * kLaP + r] = (r < kb && c < kb) ? (r >= c ? A[r + (size_t)c * lda] : 0.0)
                                         : (r == c ? 1.0 : 0.0);
    x[c * kLaP + r] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  bool bad = false;
  if (t < 32) {
    const LaBuf none{nullptr, nullptr, nullptr, nullptr};
    la_panel(a, x, none, buf(0, 0), buf(1, 0), buf(2, 0), buf(3, 0), 0, bad);
  }
  __syncthreads();
#pragma unroll 1
  for (int J = 0; J < 15; ++J) {
    TLG_PHASE(0);
    const int j = 4 * J, par = J & 1;
    const LaBuf o{buf(0, par), buf(1, par), buf(2, par), buf(3, par)};
    if (t < 32) {
      la_panel(a, x, o, buf(0, par ^ 1), buf(1, par ^ 1), buf(2, par ^ 1), buf(3, par ^ 1), j + 4,
               bad);
      TLG_PHASE(6);
    } else {
      // Items: 4-column groups x 32-row strips, lane = row.
      //   A: column groups cg >= J+2 (rows >= 4cg);   X: column groups <= J (rows >= j+8).
      const int lane = t & 31, w = (t >> 5) - 1;
      const int cgA = J + 2;
      const int nA = (16 - cgA) * 2;
      const int nX = (J + 1) * 2;
      for (int e = w; e < nA + nX; e += 3) {
        const bool isA = e < nA;
        const int f = isA ? e : e - nA;
        const int cg = isA ? cgA + (f >> 1) : (f >> 1);
        const int strip = f & 1;
        const int r = 32 * strip + lane;
        const int c0 = 4 * cg;
        const int rmin = isA ? c0 : j + 8;
        if (32 * strip + 31 < rmin) continue;  // whole strip above the region
        if (r < rmin) continue;
        double lr[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) lr[q] = o.PLr[q * 64 + r];
        double* dst = isA ? a : x;
        const double* src = isA ? o.PLc : o.PXc;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double2 u = *reinterpret_cast<const double2*>(src + (c0 + k) * 4);
          const double2 v = *reinterpret_cast<const double2*>(src + (c0 + k) * 4 + 2);
          double val = dst[(c0 + k) * kLaP + r];
          val = fma(-lr[0], u.x, val);
          val = fma(-lr[1], u.y, val);
          val = fma(-lr[2], v.x, val);
          val = fma(-lr[3], v.y, val);
          dst[(c0 + k) * kLaP + r] = val;
        }
      }
      TLG_PHASE(6);
    }
    __syncthreads();
  }
  if (t == 0 && bad) atomicOr(info, 1);
  for (int e = t; e < 64 * 64; e += 128) {
    const int r = e & 63, c = e >> 6;
    if (r < kb && c < kb && r >= c) A[r + (size_t)c * lda] = a[c * kLaP + r];
    linv[r + (size_t)c * NB] = (r >= c) ? x[c * kLaP + r] : 0.0;
  }
  __syncthreads();
}

#ifndef TLG_DIAG_TILE
#define TLG_DIAG_TILE tile_potrf_inv_la
#endif

__global__ void __launch_bounds__(128) k_potrf_coop(double* __restrict__ A, int n, int lda,
                                                    double* __restrict__ linv,
                                                    int* __restrict__ info, double* __restrict__ X,
                                                    int ldx) {
  extern __shared__ double dyn[];
  cg::grid_group grid = cg::this_grid();
  const int nt = (n + NB - 1) / NB;
  if (X) {
    // X <- I (then X = L^-1 is built alongside the factorisation)
    const size_t total = (size_t)n * n;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
         e += (size_t)gridDim.x * blockDim.x) {
      const int r = static_cast<int>(e % n), c = static_cast<int>(e / n);
      X[r + (size_t)c * ldx] = (r == c) ? 1.0 : 0.0;
    }
    grid.sync();
  }
  for (int k = 0; k < nt; ++k) {
    const int k0 = k * NB, kb = min(NB, n - k0);
    const double* lk = linv + (size_t)k * NB * NB;
    TLG_COOP_MARK(0, k);
    if (blockIdx.x == 0)
      TLG_DIAG_TILE(A + k0 + (size_t)k0 * lda, lda, kb, linv + (size_t)k * NB * NB, info, dyn);
    grid.sync();
    TLG_COOP_MARK(1, k);
    // panel: L_ik = A_ik L_kk^-T (in place; one CTA owns a tile); with X also
    // finalise block row k of L^-1: X_kj = Linv_kk X_kj, j <= k
    const int npanel = nt - k - 1, nfin = X ? k + 1 : 0;
    for (int e = blockIdx.x; e < npanel + nfin; e += gridDim.x) {
      if (e < npanel) {
        const int i = k + 1 + e;
        const int i0 = i * NB, ib = min(NB, n - i0);
        double* P = A + i0 + (size_t)k0 * lda;
        gemm_tile(GemmDesc{ib, kb, kb, P, lda, 0, lk, NB, 1, P, lda, 1.0, 0.0, 0}, 0, 0);
      } else {
        const int j = e - npanel;
        const int j0 = j * NB, jb = min(NB, n - j0);
        double* T = X + k0 + (size_t)j0 * ldx;
        gemm_tile(GemmDesc{kb, jb, kb, lk, NB, 0, T, ldx, 0, T, ldx, 1.0, 0.0, 0}, 0, 0);
      }
      __syncthreads();
    }
    grid.sync();
    TLG_COOP_MARK(2, k);
    // trailing update of the lower tiles: A_ij -= L_ik L_jk^T, k < j <= i;
    // with X: X_ij -= L_ik X_kj, i > k >= j
    const int nr = nt - k - 1;
    const int ntiles = nr * (nr + 1) / 2;
    const int nx = X ? nr * (k + 1) : 0;
    for (int e = blockIdx.x; e < ntiles + nx; e += gridDim.x) {
      if (e < ntiles) {
        int r = 0, rem = e;
        while (rem > r) {
          rem -= r + 1;
          ++r;
        }
        const int i = k + 1 + r, j = k + 1 + rem;
        const int i0 = i * NB, j0 = j * NB, ib = min(NB, n - i0), jb = min(NB, n - j0);
        gemm_tile(GemmDesc{ib, jb, kb, A + i0 + (size_t)k0 * lda, lda, 0,
                           A + j0 + (size_t)k0 * lda, lda, 1, A + i0 + (size_t)j0 * lda, lda, -1.0,
                           1.0, 0},
                  0, 0);
      } else {
        const int f = e - ntiles;
        const int i = k + 1 + f / (k + 1), j = f % (k + 1);
        const int i0 = i * NB, j0 = j * NB, ib = min(NB, n - i0), jb = min(NB, n - j0);
        gemm_tile(GemmDesc{ib, jb, kb, A + i0 + (size_t)k0 * lda, lda, 0,
                           X + k0 + (size_t)j0 * ldx, ldx, 0, X + i0 + (size_t)j0 * ldx, ldx, -1.0,
                           1.0, 0},
                  0, 0);
      }
      __syncthreads();
    }
    grid.sync();
  }
}

// ---------------------------------------------------------------------------
// 32-wide tile path for small systems (n <= kSmallN), where every step of the
// factorisation is latency-bound: a 32 x 32 DMMA tile spreads the GEMM work
// over 4x more SMs, and the diagonal tile is factored by ONE warp entirely in
// registers (lane i owns row i), so a pivot costs shfl -> rsqrt -> mul -> fma
// instead of block barriers and shared-memory round trips.
constexpr int NB32 = 32;
constexpr int kSmallN = 1024;

// C (<= 32 x 32 at tile (tm, tn)) = alpha op(A) op(B) + beta C, 128 threads;
// warp w owns the 16 x 16 quadrant (w & 1, w >> 1). uplo 2 as in gemm_tile.
__device__ __forceinline__ void gemm32_tile(const GemmDesc& d, int tm, int tn) {
  constexpr int P = 36;
  __shared__ double As32[32][P];
  __shared__ double Bs32[32][P];
  const int m0 = tm * 32, n0 = tn * 32;
  if (m0 >= d.M || n0 >= d.N) return;
  const int K = (d.uplo == 2) ? min(d.K, m0 + 32) : d.K;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int wm = (w & 1) * 16, wn = (w >> 1) * 16;
  double acc[2][2][2] = {};
  double cpre[2][2][2];
  if (d.beta != 0.0) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = m0 + wm + i * 8 + (lane >> 2), c = n0 + wn + j * 8 + 2 * (lane & 3) + h;
          cpre[i][j][h] = (r < d.M && c < d.N) ? d.C[r + (size_t)c * d.ldc] : 0.0;
        }
  }
  double pa[8], pb[8];
  // element e = t + 128 s of the 32 x 32 chunk: (k, i) = (e >> 5, e & 31) when
  // the source is contiguous along i, else (e & 31, e >> 5)
  auto fetch = [&](int k0) {
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int e = t + 128 * s, lo = e & 31, hi = e >> 5;
      if (!d.ta) {
        const int gi = m0 + lo, gk = k0 + hi;
        pa[s] = (gi < d.M && gk < K) ? d.A[gi + (size_t)gk * d.lda] : 0.0;
      } else {
        const int gk = k0 + lo, gi = m0 + hi;
        pa[s] = (gi < d.M && gk < K) ? d.A[gk + (size_t)gi * d.lda] : 0.0;
      }
      if (!d.tb) {
        const int gk = k0 + lo, gj = n0 + hi;
        pb[s] = (gj < d.N && gk < K) ? d.B[gk + (size_t)gj * d.ldb] : 0.0;
      } else {
        const int gj = n0 + lo, gk = k0 + hi;
        pb[s] = (gj < d.N && gk < K) ? d.B[gj + (size_t)gk * d.ldb] : 0.0;
      }
    }
  };
  if (K > 0) fetch(0);
  for (int k0 = 0; k0 < K; k0 += 32) {
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int e = t + 128 * s, lo = e & 31, hi = e >> 5;
      if (!d.ta) As32[hi][lo] = pa[s];
      else As32[lo][hi] = pa[s];
      if (!d.tb) Bs32[lo][hi] = pb[s];
      else Bs32[hi][lo] = pb[s];
    }
    __syncthreads();
    if (k0 + 32 < K) fetch(k0 + 32);
#pragma unroll
    for (int kk = 0; kk < 32; kk += 4) {
      double a[2], b[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) a[i] = As32[kk + (lane & 3)][wm + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = Bs32[kk + (lane & 3)][wn + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = m0 + wm + i * 8 + (lane >> 2), c = n0 + wn + j * 8 + 2 * (lane & 3) + h;
        if (r < d.M && c < d.N) {
          const double v = d.alpha * acc[i][j][h];
          d.C[r + (size_t)c * d.ldc] = (d.beta == 0.0) ? v : fma(d.beta, cpre[i][j][h], v);
        }
      }
}

// bwt: lower tile bandwidth (tile (i, j) is zero for i - j > bwt; fill-in of
// a banded matrix stays inside the band), nt - 1 for a dense matrix.
// Lookahead schedule (two grid barriers per step): the diagonal tile k+1 is
// updated and factored by block 0 inside the trailing phase of step k, while
// the other blocks apply the rest of step k's trailing update (and X's).
// Measured against a three-barrier schedule (tile k factored alone, trailing
// shared by all blocks) on one box: n=400 229 vs 243 us, n=1024 584 vs 650,
// banded n=4096 bw=700 3.0 vs 4.1 ms.
__global__ void __launch_bounds__(128) k_potrf_coop32(double* __restrict__ A, int n, int lda,
                                                      double* __restrict__ linv,
                                                      int* __restrict__ info,
                                                      double* __restrict__ X, int ldx, int bwt) {
  __shared__ double wsh[kWarpPotrfSmem];
  cg::grid_group grid = cg::this_grid();
  const int nt = (n + NB32 - 1) / NB32;
  const int G = gridDim.x, bid = blockIdx.x;
  if (X) {
    const size_t total = (size_t)n * n;
    for (size_t e = bid * (size_t)blockDim.x + threadIdx.x; e < total;
         e += (size_t)G * blockDim.x) {
      const int r = static_cast<int>(e % n), c = static_cast<int>(e / n);
      X[r + (size_t)c * ldx] = (r == c) ? 1.0 : 0.0;
    }
  }
  if (bid == 0 && threadIdx.x < 32) warp_potrf_inv32(A, lda, min(NB32, n), linv, info, wsh);
  grid.sync();
  for (int k = 0; k < nt; ++k) {
    const int k0 = k * NB32, kb = min(NB32, n - k0);
    const double* lk = linv + (size_t)k * NB32 * NB32;
    TLG_COOP_MARK(0, k);
    TLG_COOP_MARK(1, k);
    const int last = min(nt - 1, k + bwt);  // last tile row inside the band
    const int npanel = last - k, nfin = X ? k + 1 : 0;
    for (int e = bid; e < npanel + nfin; e += G) {
      if (e < npanel) {
        const int i0 = (k + 1 + e) * NB32, ib = min(NB32, n - i0);
        double* P = A + i0 + (size_t)k0 * lda;
        gemm32_tile(GemmDesc{ib, kb, kb, P, lda, 0, lk, NB32, 1, P, lda, 1.0, 0.0, 0}, 0, 0);
      } else {
        const int j0 = (e - npanel) * NB32, jb = min(NB32, n - j0);
        double* T = X + k0 + (size_t)j0 * ldx;
        gemm32_tile(GemmDesc{kb, jb, kb, lk, NB32, 0, T, ldx, 0, T, ldx, 1.0, 0.0, 0}, 0, 0);
      }
    }
    grid.sync();
    TLG_COOP_MARK(2, k);
    if (k + 1 == nt) break;
    const int nr = last - k;
    const int ntiles = nr * (nr + 1) / 2;
    const int nx = X ? nr * (k + 1) : 0;
    // trailing tile e -> (i, j) = (k + 1 + r, k + 1 + rem), rem <= r; e = 0 is
    // the next diagonal tile
    auto trailing = [&](int e) {
      if (e < ntiles) {
        int r = 0, rem = e;
        while (rem > r) {
          rem -= r + 1;
          ++r;
        }
        const int i0 = (k + 1 + r) * NB32, j0 = (k + 1 + rem) * NB32;
        const int ib = min(NB32, n - i0), jb = min(NB32, n - j0);
        gemm32_tile(GemmDesc{ib, jb, kb, A + i0 + (size_t)k0 * lda, lda, 0,
                             A + j0 + (size_t)k0 * lda, lda, 1, A + i0 + (size_t)j0 * lda, lda,
                             -1.0, 1.0, 0},
                    0, 0);
      } else {
        const int f = e - ntiles;
        const int i0 = (k + 1 + f / (k + 1)) * NB32, j0 = (f % (k + 1)) * NB32;
        const int ib = min(NB32, n - i0), jb = min(NB32, n - j0);
        gemm32_tile(GemmDesc{ib, jb, kb, A + i0 + (size_t)k0 * lda, lda, 0,
                             X + k0 + (size_t)j0 * ldx, ldx, 0, X + i0 + (size_t)j0 * ldx, ldx,
                             -1.0, 1.0, 0},
                    0, 0);
      }
    };
    if (bid == 0) {
      if (ntiles > 0) trailing(0);
      __syncthreads();
      const int k1 = (k + 1) * NB32;
      if (threadIdx.x < 32)
        warp_potrf_inv32(A + k1 + (size_t)k1 * lda, lda, min(NB32, n - k1),
                         linv + (size_t)(k + 1) * NB32 * NB32, info, wsh);
      __syncthreads();
      if (G == 1)
        for (int e = 1; e < ntiles + nx; ++e) trailing(e);
    } else {
      for (int e = bid; e < ntiles + nx; e += G - 1) trailing(e);
    }
    grid.sync();
  }
}

// Banded Cholesky solve L L^T x = b with the 32-wide factor (L in A, the
// diagonal-tile inverses in linv) as a dataflow over row blocks of kFlowRB
// rows, without grid barriers: persistent CTAs take blocks in order (forward
// ascending, backward descending), and block i waits, tile by tile, only for
// the published solution of the blocks it reads (an acquire flag per block).
// The off-diagonal band tiles of a block are summed by its 8 warps while the
// blocks ahead are still being solved, so the critical path per block is its
// last tile product, the intra-block sequence of diagonal 32-tile steps and
// one flag hand-off — about 2 us, against a grid barrier plus four
// dependent round trips per 32 rows before.
// Forward, row r of tile ti: y_ti = Linv_ti (b_ti - sum_{tj in band} L_ti,tj y_tj);
// backward: x_ti = Linv_ti^T (y_ti - sum_{tj in band} L_tj,ti^T x_tj).
constexpr int kFlowSub = 4;                // 32-row tiles per block
constexpr int kFlowRB = 32 * kFlowSub;     // rows per block
constexpr int kFlowThreads = 256;          // 8 warps: 2 per sub-tile
constexpr int kFlowW = kFlowThreads / 32;
constexpr int kFlowP = 33;                 // smem tile pitch
constexpr int kFlowIntra = kFlowSub * (kFlowSub - 1) / 2;  // off-diagonal tiles inside a block
// dynamic smem: Linv tiles + intra-block L tiles ([r][c], pitch 33), the
// block's right-hand side, per-warp partials, per-warp staged solution tiles
constexpr size_t kFlowSmem =
    sizeof(double) * ((kFlowSub + kFlowIntra) * 32 * kFlowP + kFlowRB + kFlowW * 32 + kFlowW * 2 * 32 +
                      kFlowW * 32 * kFlowP);

// Flag observation: relaxed loads (an acquire load invalidates the whole L1
// on every execution — CCTL.IVALL in the SASS), then one acquire fence once
// the awaited flags are seen. Operand data is read through L2 (__ldcg).
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// Publication: the block's (or warp's) stores, a CTA barrier (or
// __syncwarp), then one st.release by one thread — release is cumulative
// over the writes ordered before it by the barrier, so no per-thread
// __threadfence (which waited for every thread's stores to be acknowledged)
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// lane 0 waits for block `blk`, then the warp reads what it published. The
// spin uses relaxed loads; the confirming load is an acquire (not a fence:
// a fence would also wait for the lane's outstanding band-row prefetches)
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_block(const int* flag, int blk, int epoch) {
  if ((threadIdx.x & 31) == 0) {
    while (ld_relaxed(flag + blk) != epoch) {
    }
    (void)ld_acquire(flag + blk);
  }
  __syncwarp();
}

// sum over lanes of v[c] for all 32 c at once (recursive halving, 31
// shuffles): lane c returns sum_lanes v[c]
__device__ __forceinline__ double warp_transpose_sum(double (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int h = 16; h > 0; h >>= 1) {
    const bool up = lane & h;
#pragma unroll
    for (int q = 0; q < h; ++q) {
      const double send = up ? v[q] : v[q + h];
      const double keep = up ? v[q + h] : v[q];
      v[q] = keep + __shfl_xor_sync(0xffffffffu, send, h);
    }
  }
  return v[0];
}

#ifdef TLG_FLOW_TRACE
// Diagnostics build only (tools/band_trace.py): globaltimer stamps of forward
// band-solve blocks [kBt0, kBt0 + 64)
constexpr int kBt0 = 300;
__device__ unsigned long long tlg_band_trace[64][8];
__device__ unsigned long long tlg_band_trace_b[64][8];
__device__ __forceinline__ unsigned long long gtime_b() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
  return v;
}
#define TLG_BT(blk, slot) \
  do { if (threadIdx.x == 0 && (blk) >= kBt0 && (blk) < kBt0 + 64) tlg_band_trace[(blk) - kBt0][slot] = gtime_b(); } while (0)
#define TLG_BTB(q, slot) \
  do { if (threadIdx.x == 0 && (q) >= kBt0 && (q) < kBt0 + 64) tlg_band_trace_b[(q) - kBt0][slot] = gtime_b(); } while (0)
__device__ __forceinline__ unsigned long long gtime_dep(double dep) {
  unsigned long long v;
  asm volatile("{\n .reg .f64 t;\n mov.f64 t, %1;\n mov.u64 %0, %globaltimer;\n}" : "=l"(v) : "d"(dep));
  return v;
}
#define TLG_BTBD(q, slot, dep) \
  do { const double _d = (dep); if (threadIdx.x == 0 && (q) >= kBt0 && (q) < kBt0 + 64) tlg_band_trace_b[(q) - kBt0][slot] = gtime_dep(_d); } while (0)
extern "C" int tlg_debug_band_trace(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, tlg_band_trace, sizeof(tlg_band_trace)) != cudaSuccess) return 1;
  return cudaMemcpyFromSymbol(out + 64 * 8, tlg_band_trace_b, sizeof(tlg_band_trace_b)) == cudaSuccess ? 0 : 1;
}
#else
#define TLG_BT(blk, slot)
#define TLG_BTB(q, slot)
#define TLG_BTBD(q, slot, dep)
#endif

// sum_c a[c] b[c] over 32 terms as four interleaved chains (the band
// solve's per-block steps are latency-bound: a 32-long FMA chain is ~260
// cycles, four chains of 8 ~70)
template <class FA, class FB>
__device__ __forceinline__ double dot32x4(FA a, FB b) {
  double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int c = 0; c < 32; ++c) s[c & 3] = fma(a(c), b(c), s[c & 3]);
  return (s[0] + s[1]) + (s[2] + s[3]);
}

// the same through a per-warp [32][33] shared buffer: 32 stores, 32 loads
// (the 31-round shuffle version measured ~8 us per call inside the backward
// band solve's critical section)
__device__ __forceinline__ double warp_transpose_sum_smem(const double (&v)[32], double* buf) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < 32; ++c) buf[lane * 33 + c] = v[c];
  __syncwarp();
  double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int r = 0; r < 32; ++r) s[r & 3] += buf[r * 33 + lane];
  __syncwarp();
  return (s[0] + s[1]) + (s[2] + s[3]);
}

// Stages block [t0, t1)'s diagonal inverses (lower kb x kb part) and its
// off-diagonal tiles L(tr, tc), t0 <= tc < tr < t1, in the band, as [r][c].
__device__ __forceinline__ void flow_stage(const double* __restrict__ L, int n, int ld, int bwt,
                                           const double* __restrict__ linv, int t0, int t1,
                                           double* sLi, double* sT) {
  for (int e = threadIdx.x; e < kFlowSub * 1024; e += kFlowThreads) {
    const int s = e >> 10, r = e & 31, c = (e >> 5) & 31, ti = t0 + s;
    double v = 0.0;
    if (ti < t1 && c <= r && ti * 32 + r < n) v = linv[(size_t)ti * 1024 + r + 32 * c];
    sLi[(s * 32 + r) * kFlowP + c] = v;
  }
  for (int e = threadIdx.x; e < kFlowIntra * 1024; e += kFlowThreads) {
    const int q = e >> 10, r = e & 31, c = (e >> 5) & 31;
    int tr = 1, tc = 0, k = q;  // q -> (tr, tc) in (1,0), (2,0), (2,1), (3,0), ...
    while (k >= tr) {
      k -= tr;
      ++tr;
    }
    tc = k;
    const int gr = (t0 + tr) * 32 + r, gc = (t0 + tc) * 32 + c;
    double v = 0.0;
    if (t0 + tr < t1 && tr - tc <= bwt && gr < n) v = L[gr + (size_t)gc * ld];
    sT[(q * 32 + r) * kFlowP + c] = v;
  }
}
__device__ __forceinline__ int flow_intra(int tr, int tc) { return tr * (tr - 1) / 2 + tc; }

__global__ void __launch_bounds__(kFlowThreads) k_band_fwd_flow(const double* __restrict__ L, int n,
                                                                int ld, int bwt,
                                                                const double* __restrict__ linv,
                                                                const double* __restrict__ b,
                                                                double* __restrict__ y,
                                                                int* __restrict__ flag, int epoch) {
  extern __shared__ __align__(16) double fsm[];
  double* sLi = fsm;
  double* sT = sLi + kFlowSub * 32 * kFlowP;
  double* bb = sT + kFlowIntra * 32 * kFlowP;
  double* part = bb + kFlowRB;      // [warp][32]
  double* ys = part + kFlowW * 32;  // [warp][2][32]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = warp >> 1, half = warp & 1;  // this warp's sub-tile, and its half of the tiles
  const int nt = (n + 31) / 32, nb = (n + kFlowRB - 1) / kFlowRB;
  for (int i = blockIdx.x; i < nb; i += gridDim.x) {
    const int t0 = i * kFlowSub, t1 = min(nt, t0 + kFlowSub);
    const int ti = t0 + s, r = ti * 32 + lane;
    const bool row_ok = ti < t1 && r < n;
    // this block's right-hand side, loaded now (off the critical path)
    const int rb = t0 * 32 + threadIdx.x;
    const double bv = (threadIdx.x < kFlowRB && rb < n) ? b[rb] : 0.0;
    TLG_BT(i, 0);
    flow_stage(L, n, ld, bwt, linv, t0, t1, sLi, sT);
    // blocks <= i-2 (published earlier): tiles of the row's band, oldest first
    const int tlo = max(0, ti - bwt), tcrit = max(0, t0 - 2 * kFlowSub);
    double acc = 0.0;
    for (int tj = tlo + half; tj < tcrit; tj += 2) {
      wait_block(flag, tj / kFlowSub, epoch);
      ys[(warp * 2) * 32 + lane] = __ldcg(y + tj * 32 + lane);
      __syncwarp();
      if (row_ok) {
        const double* lr = L + r + (size_t)tj * 32 * ld;
        double lv[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) lv[c] = lr[(size_t)c * ld];
        const double* yw = ys + (warp * 2) * 32;
        acc += dot32x4([&](int c) { return lv[c]; }, [&](int c) { return yw[c]; });
      }
      __syncwarp();
    }
    // blocks i-2 and i-1 (the last two hand-offs): each block's tile rows are
    // loaded before its wait (the waits are acquire loads, which do not wait
    // for them), so only the y loads and the products follow a flag
    auto crit_block = [&](int blk) {
      const int tb = blk * kFlowSub;
      double lv[2][32];
      int tjs[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int tj = tb + half + 2 * u;
        tjs[u] = (tj < t0 && tj >= tlo && row_ok) ? tj : -1;
        const double* lr = L + (row_ok ? r : 0) + (size_t)max(tj, 0) * 32 * ld;
#pragma unroll
        for (int c = 0; c < 32; ++c) lv[u][c] = tjs[u] >= 0 ? lr[(size_t)c * ld] : 0.0;
      }
      if (blk == i - 1) TLG_BT(i, 1);
      wait_block(flag, blk, epoch);
      if (blk == i - 1) TLG_BT(i, 2);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int tj = tb + half + 2 * u;
        ys[(warp * 2 + u) * 32 + lane] = (tj < t0 && tj >= tlo) ? __ldcg(y + tj * 32 + lane) : 0.0;
      }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (tjs[u] >= 0) {
          const double* yw = ys + (warp * 2 + u) * 32;
          acc += dot32x4([&](int c) { return lv[u][c]; }, [&](int c) { return yw[c]; });
        }
      __syncwarp();
    };
    if (i > 1) crit_block(i - 2);
    if (i > 0) crit_block(i - 1);
    part[warp * 32 + lane] = acc;
    __syncthreads();
    if (threadIdx.x < kFlowRB) {
      const int q = threadIdx.x >> 5, rr = t0 * 32 + threadIdx.x;
      bb[threadIdx.x] = rr < n ? bv - (part[(2 * q) * 32 + lane] + part[(2 * q + 1) * 32 + lane]) : 0.0;
    }
    __syncthreads();
    TLG_BT(i, 3);
    // the block's own tiles, in order (all operands in shared memory)
    for (int tk = t0; tk < t1; ++tk) {
      const int k = tk - t0;
      if (warp == 0) {
        const double* li = sLi + (k * 32 + lane) * kFlowP;
        const double* bk = bb + k * 32;
        const double v = dot32x4([&](int c) { return li[c]; }, [&](int c) { return bk[c]; });
        const int rr = tk * 32 + lane;
        if (rr < n) y[rr] = v;
        bb[k * 32 + lane] = rr < n ? v : 0.0;
      }
      __syncthreads();
      const int tr = tk + 1 + warp;
      if (tr < t1 && tr - tk <= bwt) {
        const double* tl = sT + (flow_intra(tr - t0, k) * 32 + lane) * kFlowP;
        const double* bk = bb + k * 32;
        const double a = dot32x4([&](int c) { return tl[c]; }, [&](int c) { return bk[c]; });
        bb[(tr - t0) * 32 + lane] -= a;
      }
      __syncthreads();
    }
    TLG_BT(i, 4);
    __syncthreads();
    if (threadIdx.x == 0) st_release(flag + i, epoch);
    TLG_BT(i, 5);
  }
}

__global__ void __launch_bounds__(kFlowThreads) k_band_bwd_flow(const double* __restrict__ L, int n,
                                                                int ld, int bwt,
                                                                const double* __restrict__ linv,
                                                                const double* __restrict__ y,
                                                                double* __restrict__ x,
                                                                int* __restrict__ flag, int epoch) {
  extern __shared__ __align__(16) double fsm[];
  double* sLi = fsm;
  double* sT = sLi + kFlowSub * 32 * kFlowP;
  double* bb = sT + kFlowIntra * 32 * kFlowP;
  double* part = bb + kFlowRB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* tbuf = part + kFlowW * 32 + kFlowW * 2 * 32 + warp * 32 * kFlowP;  // transpose-sum buffer
  const int s = warp >> 1, half = warp & 1;
  const int nt = (n + 31) / 32, nb = (n + kFlowRB - 1) / kFlowRB;
  for (int q = blockIdx.x; q < nb; q += gridDim.x) {
    const int i = nb - 1 - q;
    const int t0 = i * kFlowSub, t1 = min(nt, t0 + kFlowSub);
    const int ti = t0 + s;  // column tile of this warp's sub-tile
    const int rb = t0 * 32 + threadIdx.x;  // this block's y, loaded off the critical path
    const double yv = (threadIdx.x < kFlowRB && rb < n) ? y[rb] : 0.0;
    TLG_BTB(q, 0);
    flow_stage(L, n, ld, bwt, linv, t0, t1, sLi, sT);
    // v[c] accumulates sum_r L(tj r, ti c) x(tj r) over this warp's tiles
    // (lane = r); one transpose-sum at the end
    double v[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = 0.0;
    const int thi = ti < t1 ? min(nt - 1, ti + bwt) : -1;  // last tile of the column's band
    const int tcrit = t1 + 2 * kFlowSub;                    // tiles of blocks i+1, i+2: [t1, tcrit)
    // blocks >= i+3, oldest (farthest) first
    for (int tj = thi - half; tj >= tcrit; tj -= 2) {
      wait_block(flag, nb - 1 - tj / kFlowSub, epoch);
      const int r = tj * 32 + lane;
      const double xr = r < n ? __ldcg(x + r) : 0.0;
      const double* lr = L + min(r, n - 1) + (size_t)ti * 32 * ld;
#pragma unroll
      for (int c = 0; c < 32; ++c) v[c] = fma(r < n ? lr[(size_t)c * ld] : 0.0, xr, v[c]);
    }
    // blocks i+2 and i+1 (the last two hand-offs): tile rows loaded before
    // each block's wait, then the x loads and the products
    auto crit_block = [&](int bi) {
      const int tb = bi * kFlowSub;
      double lv[2][32];
      int tjs[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int tj = tb + half + 2 * u;
        const int r = tj * 32 + lane;
        tjs[u] = (tj <= thi && tj < tb + kFlowSub && tj < nt) ? tj : -1;
        const double* lr = L + min(max(r, 0), n - 1) + (size_t)max(ti, 0) * 32 * ld;
#pragma unroll
        for (int c = 0; c < 32; ++c) lv[u][c] = (tjs[u] >= 0 && r < n) ? lr[(size_t)c * ld] : 0.0;
      }
      if (bi == i + 1) TLG_BTB(q, 1);
      wait_block(flag, nb - 1 - bi, epoch);
      if (bi == i + 1) TLG_BTB(q, 2);
      double xr[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int r = tjs[u] * 32 + lane;
        xr[u] = (tjs[u] >= 0 && r < n) ? __ldcg(x + r) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = fma(lv[u][c], xr[u], v[c]);
    };
    if (i + 2 < nb) crit_block(i + 2);
    if (i + 1 < nb) crit_block(i + 1);
    TLG_BTBD(q, 6, v[0] + v[31]);
    const double vsum = warp_transpose_sum_smem(v, tbuf);
    TLG_BTBD(q, 7, vsum);
    part[warp * 32 + lane] = vsum;
    __syncthreads();
    if (threadIdx.x < kFlowRB) {
      const int qq = threadIdx.x >> 5, rr = t0 * 32 + threadIdx.x;
      bb[threadIdx.x] = rr < n ? yv - (part[(2 * qq) * 32 + lane] + part[(2 * qq + 1) * 32 + lane]) : 0.0;
    }
    __syncthreads();
    TLG_BTB(q, 3);
    for (int tk = t1 - 1; tk >= t0; --tk) {
      const int k = tk - t0;
      if (warp == 0) {
        // x_tk = Linv^T z: lane c reads column c of the staged inverse
        const double* lc = sLi + k * 32 * kFlowP + lane;
        const double* bk = bb + k * 32;
        const double a = dot32x4([&](int rr) { return lc[rr * kFlowP]; }, [&](int rr) { return bk[rr]; });
        const int c = tk * 32 + lane;
        if (c < n) x[c] = a;
        bb[k * 32 + lane] = c < n ? a : 0.0;
      }
      __syncthreads();
      const int tc = tk - 1 - warp;  // z_tc -= L(tk, tc)^T x_tk
      if (tc >= t0 && tk - tc <= bwt) {
        const double* tl = sT + flow_intra(k, tc - t0) * 32 * kFlowP + lane;
        const double* bk = bb + k * 32;
        const double a = dot32x4([&](int rr) { return tl[rr * kFlowP]; }, [&](int rr) { return bk[rr]; });
        bb[(tc - t0) * 32 + lane] -= a;
      }
      __syncthreads();
    }
    TLG_BTB(q, 4);
    __syncthreads();
    if (threadIdx.x == 0) st_release(flag + q, epoch);
    TLG_BTB(q, 5);
  }
}

void band_solve(tlg_ctx* ctx, const double* L, int n, int ld, int band, double* b) {
  if (n <= 0) return;
  require(ctx->linv32_owner == L, TLG_RUNTIME_ERROR, "band_solve: matrix was not factored last");
  const int nt = (n + NB32 - 1) / NB32;
  int bwt = std::min(nt - 1, (std::max(band, 0) + NB32 - 1) / NB32);
  const double* linv = ctx->ws<double>(S_LINV, 1);
  double* y = ctx->ws<double>(S_XINV2, n);
  double* x = ctx->ws<double>(S_BSOLVE, n);
  const int nb = (n + kFlowRB - 1) / kFlowRB;
  int* flags = ctx->ws<int>(S_FLOWFLAG, 2 * static_cast<size_t>(nb));
  TLG_CUDA(cudaMemsetAsync(flags, 0, 2 * static_cast<size_t>(nb) * sizeof(int), ctx->stream));
  int epoch = 1;
  // every CTA co-resident (cooperative launch): a waiting block's producers
  // are always running
  // one CTA per SM: fewer pollers, and a CTA's next block is far behind the
  // wavefront anyway
  const int g1 = std::max(1, std::min(nb, ctx->num_sms));
  const int g2 = g1;
  int* f1 = flags;
  int* f2 = flags + nb;
  TLG_CUDA(cudaFuncSetAttribute(k_band_fwd_flow, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kFlowSmem)));
  TLG_CUDA(cudaFuncSetAttribute(k_band_bwd_flow, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kFlowSmem)));
  void* a1[] = {&L, &n, &ld, &bwt, &linv, &b, &y, &f1, &epoch};
  TLG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_band_fwd_flow), dim3(g1),
                                       dim3(kFlowThreads), a1, kFlowSmem, ctx->stream));
  ++ctx->launches;
  void* a2[] = {&L, &n, &ld, &bwt, &linv, &y, &x, &f2, &epoch};
  TLG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_band_bwd_flow), dim3(g2),
                                       dim3(kFlowThreads), a2, kFlowSmem, ctx->stream));
  ++ctx->launches;
  TLG_CUDA(cudaMemcpyAsync(b, x, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToDevice, ctx->stream));
}

// B <- L^-1 B (trans = 0) or L^-T B (trans = 1), one CTA per 64-column slab
// of B walking the tile rows: B_k -= L_kj X_j (DMMA), X_k = Linv_kk B_k.
__global__ void __launch_bounds__(128) k_trsm_tiles(const double* __restrict__ L, int n, int ldl,
                                                    const double* __restrict__ linv,
                                                    double* __restrict__ B, int nrhs, int ldb,
                                                    int trans) {
  const int c0 = blockIdx.x * NB, nb = min(NB, nrhs - c0);
  const int nt = (n + NB - 1) / NB;
  double* Bc = B + (size_t)c0 * ldb;
  for (int s = 0; s < nt; ++s) {
    const int k = trans ? nt - 1 - s : s;
    const int k0 = k * NB, kb = min(NB, n - k0);
    if (!trans) {
      if (k0 > 0)
        gemm_tile(GemmDesc{kb, nb, k0, L + k0, ldl, 0, Bc, ldb, 0, Bc + k0, ldb, -1.0, 1.0, 0}, 0,
                  0);
    } else {
      const int rest = n - k0 - kb;
      if (rest > 0)
        gemm_tile(GemmDesc{kb, nb, rest, L + (k0 + kb) + (size_t)k0 * ldl, ldl, 1, Bc + k0 + kb, ldb,
                           0, Bc + k0, ldb, -1.0, 1.0, 0},
                  0, 0);
    }
    __syncthreads();
    gemm_tile(GemmDesc{kb, nb, kb, linv + (size_t)k * NB * NB, NB, trans, Bc + k0, ldb, 0, Bc + k0,
                       ldb, 1.0, 0.0, 0},
              0, 0);
    __syncthreads();
  }
}

// Banded / dense 32-wide Cholesky as a task dataflow (no grid barriers).
// Task (i, j) owns band tile (i, j): it applies its updates
// A_ij -= L_ik L_jk^T for k = max(0, i - bwt) .. j - 1 in ascending k (so the
// result is bit-reproducible), waiting per k for the two operand tiles'
// "final" flags, then finalises the tile — the one-warp Cholesky + inverse
// when i == j, L_ij = A_ij Linv_j^T (after tile (j, j)) otherwise — and
// publishes it. Persistent CTAs claim tasks from a counter in column-major
// order; every wait targets an earlier-claimed task and all CTAs are
// co-resident, so the schedule cannot deadlock. Columns overlap freely: the
// critical path per column is the diagonal chain POTRF(j-1) -> TRSM(j, j-1)
// -> last update of (j, j) -> POTRF(j), while the bulk of the updates runs
// ahead of it.
#ifndef TLG_PF_MINB
#define TLG_PF_MINB 3
#endif
#ifdef TLG_FLOW_TRACE
// Diagnostics build only (tools/flow_trace.py): globaltimer stamps of the
// diagonal and first-solve tasks of columns [kTr0, kTr0 + kTrN).
constexpr int kTr0 = 1000, kTrN = 64;
__device__ unsigned long long tlg_flow_trace[kTrN][8];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
  return v;
}
#define TLG_TR(col, slot) \
  do { if (t == 0 && (col) >= kTr0 && (col) < kTr0 + kTrN) tlg_flow_trace[(col) - kTr0][slot] = gtime(); } while (0)
__device__ unsigned long long tlg_flow_trace2[kTrN][8];
#define TLG_TRW(col, slot) \
  do { if ((col) >= kTr0 && (col) < kTr0 + kTrN) tlg_flow_trace2[(col) - kTr0][slot] = gtime(); } while (0)
#else
#define TLG_TR(col, slot)
#define TLG_TRW(col, slot)
#endif
#ifndef TLG_SPIN_NS
#define TLG_SPIN_NS 64
#endif
#if TLG_SPIN_NS > 0
#define TLG_SPIN_PAUSE __nanosleep(TLG_SPIN_NS)
#else
#define TLG_SPIN_PAUSE
#endif
constexpr int kPFP = 36;  // smem tile pitch (conflict-free fragments, as gemm32_tile)

__global__ void __launch_bounds__(128, TLG_PF_MINB) k_potrf_flow32(double* __restrict__ A, int n, int lda, int bwt,
                                                      double* __restrict__ linv, int* __restrict__ info,
                                                      double* __restrict__ X, int ldx,
                                                      int* __restrict__ flag,
                                                      unsigned long long* __restrict__ counter,
                                                      int epoch, const int2* __restrict__ order) {
  __shared__ __align__(16) double Xs[2][32][kPFP];  // double-buffered operand tiles
  __shared__ __align__(16) double Ys[2][32][kPFP];
  static_assert(2 * 32 * kPFP >= kWarp2PotrfSmem, "diagonal-factor scratch aliases Xs");
  double* wsh = &Xs[0][0][0];  // the diagonal factor's scratch (Xs is idle then)
  __shared__ long long task_s;
  __shared__ int s_first;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int wm = (w & 1) * 16, wn = (w >> 1) * 16;
  const int nt = (n + 31) / 32;
  const long long T0 = static_cast<long long>(nt - bwt) * (bwt + 1);
  const long long total = T0 + static_cast<long long>(bwt) * (bwt + 1) / 2;
  auto fl = [&](int i, int j) { return flag + static_cast<size_t>(j) * (bwt + 1) + (i - j); };
  // X = L^-1 tasks (when X != nullptr) follow all factor tasks: tile (i, j),
  // i >= j, row-major; xfl(i, j) its flag
  int* xflag = flag + static_cast<size_t>(nt) * (bwt + 1);
  auto xfl = [&](int i, int j) { return xflag + static_cast<size_t>(j) * nt + i; };
  const long long total_all = total + (X ? static_cast<long long>(nt) * (nt + 1) / 2 : 0);
  const bool async_ok = (lda % 2 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0);
  auto spin = [&](const int* f) {
    while (ld_relaxed(f) != epoch) TLG_SPIN_PAUSE;
  };
  for (;;) {
    if (t == 0) task_s = static_cast<long long>(atomicAdd(counter, 1ull));
    __syncthreads();
    const long long task = task_s;
    __syncthreads();
    if (task >= total_all) break;
    // with a claim-order table, entry (i, j) is factor task (i, j) and
    // (i, -1 - j) is L^-1 task (i, j)
    int2 oij = make_int2(0, 0);
    if (order) oij = order[task];
    if (order ? oij.y < 0 : task >= total) {
      // ---- X_ij = -Linv_i sum_{k = max(j, i - bwt)}^{i-1} L_ik X_kj  (X_jj = Linv_j)
      // row-major over the lower tiles: row i's tiles depend on earlier rows
      // only, so the rows form a wavefront with every column in flight
      int i, j;
      if (order) {
        i = oij.x;
        j = -1 - oij.y;
      } else {
        const long long r = task - total;
        i = static_cast<int>((sqrt(8.0 * static_cast<double>(r) + 1.0) - 1.0) * 0.5);
        while (static_cast<long long>(i) * (i + 1) / 2 > r) --i;
        while (static_cast<long long>(i + 1) * (i + 2) / 2 <= r) ++i;
        j = static_cast<int>(r - static_cast<long long>(i) * (i + 1) / 2);
      }
      const int i0 = i * 32, j0 = j * 32, ib = min(32, n - i0), jb = min(32, n - j0);
      if (i == j) {
        if (t == 0) {
          spin(fl(j, j));
          (void)ld_acquire(fl(j, j));
        }
        __syncthreads();
        const double* lj = linv + static_cast<size_t>(j) * 1024;
        for (int e = t; e < 1024; e += 128) {
          const int rr = e & 31, c = e >> 5;
          if (rr < jb && c < jb) X[(j0 + rr) + static_cast<size_t>(j0 + c) * ldx] = c <= rr ? __ldcg(lj + e) : 0.0;
        }
      } else {
        double acc[2][2][2] = {};
        // operands of step k in registers (element e = t + 128 s: a = e & 31
        // along the contiguous dimension, b = e >> 5), prefetched one step
        // ahead; readiness from one relaxed sweep of the remaining flags
        double xa[8], xb[8];
        auto xfetch = [&](int k) {
          const int k0 = k * 32;
#pragma unroll
          for (int s2 = 0; s2 < 8; ++s2) {
            const int e = t + 128 * s2, a = e & 31, b = e >> 5;
            xa[s2] = (i0 + a < n && k0 + b < n) ? __ldcg(A + (i0 + a) + static_cast<size_t>(k0 + b) * lda) : 0.0;
            xb[s2] = (k0 + a < n && j0 + b < n) ? __ldcg(X + (k0 + a) + static_cast<size_t>(j0 + b) * ldx) : 0.0;
          }
        };
        auto xstash = [&](int bf) {
#pragma unroll
          for (int s2 = 0; s2 < 8; ++s2) {
            const int e = t + 128 * s2;
            Xs[bf][e >> 5][e & 31] = xa[s2];  // Xs[q][r] = L(i0 + r, k0 + q)
            Ys[bf][e >> 5][e & 31] = xb[s2];  // Ys[c][q] = X(k0 + q, j0 + c)
          }
        };
        const int kl = max(j, i - bwt);
        auto x_first_unready = [&](int from) {
          if (t == 0) s_first = i;
          __syncthreads();
          for (int kk = from + t; kk < i; kk += 128)
            if (ld_relaxed(fl(i, kk)) != epoch || ld_relaxed(xfl(kk, j)) != epoch) atomicMin(&s_first, kk);
          fence_acquire();
          __syncthreads();
          const int f = s_first;
          __syncthreads();
          return f;
        };
        int xready = x_first_unready(kl);
        auto xensure = [&](int k) {
          if (k < xready) return;
          if (t == 0) {
            spin(fl(i, k));
            spin(xfl(k, j));
            (void)ld_acquire(fl(i, k));
            (void)ld_acquire(xfl(k, j));
          }
          __syncthreads();
          xready = max(k + 1, x_first_unready(k + 1));
        };
        xensure(kl);
        xfetch(kl);
        xstash(kl & 1);
        __syncthreads();
        for (int k = kl; k < i; ++k) {
          const bool more = k + 1 < i;
          if (more) {
            xensure(k + 1);
            xfetch(k + 1);
          }
          const int bf = k & 1;
#pragma unroll
          for (int kk = 0; kk < 32; kk += 4) {
            double av[2], bv[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) av[q] = Xs[bf][kk + (lane & 3)][wm + q * 8 + (lane >> 2)];
#pragma unroll
            for (int q = 0; q < 2; ++q) bv[q] = Ys[bf][wn + q * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
            for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
              for (int b2 = 0; b2 < 2; ++b2) dmma(acc[a2][b2][0], acc[a2][b2][1], av[a2], bv[b2]);
          }
          if (more) xstash(bf ^ 1);
          __syncthreads();
        }
        if (t == 0) {
          spin(fl(i, i));
          (void)ld_acquire(fl(i, i));
        }
        // Xs[q][r] = Linv_i(r, q), Ys[q][c] = acc(q, c)
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int rr = wm + a * 8 + (lane >> 2), c = wn + b * 8 + 2 * (lane & 3) + h;
              Ys[0][rr][c] = acc[a][b][h];
              acc[a][b][h] = 0.0;
            }
        __syncthreads();
        const double* li = linv + static_cast<size_t>(i) * 1024;
        for (int e = t; e < 1024; e += 128) {
          const int rr = e & 31, q = e >> 5;
          Xs[0][q][rr] = q <= rr ? __ldcg(li + e) : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 32; kk += 4) {
          double av[2], bv[2];
#pragma unroll
          for (int q = 0; q < 2; ++q) av[q] = -Xs[0][kk + (lane & 3)][wm + q * 8 + (lane >> 2)];
#pragma unroll
          for (int q = 0; q < 2; ++q) bv[q] = Ys[0][kk + (lane & 3)][wn + q * 8 + (lane >> 2)];
#pragma unroll
          for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
            for (int b2 = 0; b2 < 2; ++b2) dmma(acc[a2][b2][0], acc[a2][b2][1], av[a2], bv[b2]);
        }
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int rr = wm + a * 8 + (lane >> 2), c = wn + b * 8 + 2 * (lane & 3) + h;
              if (rr < ib && c < jb) X[(i0 + rr) + static_cast<size_t>(j0 + c) * ldx] = acc[a][b][h];
            }
      }
      __syncthreads();
      if (t == 0) st_release(xfl(i, j), epoch);
      continue;
    }
    int i, j;
    if (order) {
      i = oij.x;
      j = oij.y;
    } else if (task < T0) {
      j = static_cast<int>(task / (bwt + 1));
      i = j + static_cast<int>(task % (bwt + 1));
    } else {
      long long r = task - T0;
      j = nt - bwt;
      while (r >= nt - j) {
        r -= nt - j;
        ++j;
      }
      i = j + static_cast<int>(r);
    }
    const int i0 = i * 32, j0 = j * 32, ib = min(32, n - i0), jb = min(32, n - j0);
    if (i == j) TLG_TR(j, 0);
    if (i == j + 1) TLG_TR(j, 3);
    double acc[2][2][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = wm + a * 8 + (lane >> 2), c = wn + b * 8 + 2 * (lane & 3) + h;
          acc[a][b][h] = (r < ib && c < jb) ? A[(i0 + r) + static_cast<size_t>(j0 + c) * lda] : 0.0;
        }
    // operand rows: element e = t + 128 s of a tile, (q, r) = (e >> 5, e & 31)
    double pa[8], pb[8];
    auto fetch = [&](int k) {
      const int k0 = k * 32;
#pragma unroll
      for (int s2 = 0; s2 < 8; ++s2) {
        const int e = t + 128 * s2, r = e & 31, q = e >> 5;
        const bool qk = k0 + q < n;
        pa[s2] = (i0 + r < n && qk) ? __ldcg(A + (i0 + r) + static_cast<size_t>(k0 + q) * lda) : 0.0;
        pb[s2] = (j0 + r < n && qk) ? __ldcg(A + (j0 + r) + static_cast<size_t>(k0 + q) * lda) : 0.0;
      }
    };
    auto stash = [&](int buf) {
#pragma unroll
      for (int s2 = 0; s2 < 8; ++s2) {
        const int e = t + 128 * s2;
        Xs[buf][e >> 5][e & 31] = pa[s2];
        Ys[buf][e >> 5][e & 31] = pb[s2];
      }
    };
    // Asynchronous operand copy (cp.async, LDGSTS: global -> shared without
    // registers) when rows pair into 16-byte chunks (even lda): chunk
    // c = t + 128 s covers rows 2 (c & 15), 2 (c & 15) + 1 of column c >> 4;
    // rows past n are zero-filled.
    auto fetch_async = [&](int k, int buf) {
      const int k0 = k * 32;
#pragma unroll
      for (int s2 = 0; s2 < 8; ++s2) {
        const int c = t + 128 * s2, tile = c >> 9, q = (c >> 4) & 31, r = 2 * (c & 15);
        const int row = (tile ? j0 : i0) + r;
        const int bytes = k0 + q < n ? 8 * max(0, min(2, n - row)) : 0;
        const double* src = A + (bytes ? row + static_cast<size_t>(k0 + q) * lda : 0);
        double* dst = tile ? &Ys[buf][q][r] : &Xs[buf][q][r];
        const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(bytes)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    auto wait_async = [&]() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); };
    // Operand readiness: one parallel sweep of the flags of all remaining k
    // (one round trip) gives the first k not yet final; k below it need no
    // further polling.
    auto first_unready = [&](int from) {
      if (t == 0) s_first = j;
      __syncthreads();
      for (int kk = from + t; kk < j; kk += 128)
        if (ld_relaxed(fl(i, kk)) != epoch || ld_relaxed(fl(j, kk)) != epoch) atomicMin(&s_first, kk);
      fence_acquire();
      __syncthreads();
      const int f = s_first;
      __syncthreads();
      return f;
    };
    const int klo = max(0, i - bwt);
    int ready_end = klo < j ? first_unready(klo) : j;
    auto ensure = [&](int k) {
      if (k < ready_end) return;
      if (t == 0) {
        // acquire loads, not a fence: a fence would also wait for this
        // thread's outstanding operand copies
        while (ld_relaxed(fl(i, k)) != epoch) TLG_SPIN_PAUSE;
        while (ld_relaxed(fl(j, k)) != epoch) TLG_SPIN_PAUSE;
        (void)ld_acquire(fl(i, k));
        (void)ld_acquire(fl(j, k));
      }
      __syncthreads();
      ready_end = max(k + 1, first_unready(k + 1));
    };
    if (klo < j) {
      ensure(klo);
      if (async_ok) {
        fetch_async(klo, klo & 1);
        wait_async();
      } else {
        fetch(klo);
        stash(klo & 1);
      }
    }
    __syncthreads();
    for (int k = klo; k < j; ++k) {
      const bool more = k + 1 < j;
      if (more) {
        ensure(k + 1);
        // in flight during the products below
        if (async_ok) fetch_async(k + 1, (k + 1) & 1);
        else fetch(k + 1);
      }
      const int bf = k & 1;
#pragma unroll
      for (int kk = 0; kk < 32; kk += 4) {
        double a[2], b[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) a[q] = -Xs[bf][kk + (lane & 3)][wm + q * 8 + (lane >> 2)];
#pragma unroll
        for (int q = 0; q < 2; ++q) b[q] = Ys[bf][kk + (lane & 3)][wn + q * 8 + (lane >> 2)];
#pragma unroll
        for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
          for (int b2 = 0; b2 < 2; ++b2) dmma(acc[a2][b2][0], acc[a2][b2][1], a[a2], b[b2]);
      }
      if (more) {
        if (async_ok) wait_async();
        else stash(bf ^ 1);
      }
      __syncthreads();
    }
    if (i == j) TLG_TR(j, 1);
    if (i == j + 1) TLG_TR(j, 4);
    if (i == j) {
      // the diagonal step is the per-column critical path: the tile stays in
      // shared memory (Ys[0]) for the one-warp factor + inverse, warp 0
      // publishes Linv_j as soon as it is written (the consumers — the
      // column's solves and the L^-1 tasks — read only Linv_j), and L_jj
      // goes back to the band afterwards
      double* T = &Ys[0][0][0];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = wm + a * 8 + (lane >> 2), c = wn + b * 8 + 2 * (lane & 3) + h;
            if (c <= r) T[r + c * kPFP] = acc[a][b][h];
          }
      if (t == 0) *warp2_potrf_pub(wsh) = 0;
      __syncthreads();
      if (w < 2) {
        // warp 0 factors, warp 1 forms Linv_j one published column behind it
        TLG_TR(j, 7);
        warp2b_potrf_inv32(T, kPFP, jb, linv + static_cast<size_t>(j) * 1024, info, wsh);
        if (w == 1) {
          if (lane == 0) TLG_TRW(j, 5);
          __syncwarp();
          if (lane == 0) st_release(fl(j, j), epoch);
          if (lane == 0) TLG_TRW(j, 2);  // flag released (trace2 slot 2)
        }
      }
      __syncthreads();
      for (int e = t; e < 1024; e += 128) {
        const int r = e & 31, c = e >> 5;
        if (r < jb && c < jb && c <= r) A[(j0 + r) + static_cast<size_t>(j0 + c) * lda] = T[r + c * kPFP];
      }
      __syncthreads();  // T is reused by the next task
      continue;
    } else {
      if (t == 0) {
        while (ld_relaxed(fl(j, j)) != epoch) TLG_SPIN_PAUSE;
        (void)ld_acquire(fl(j, j));
      }
      if (i == j + 1) TLG_TR(j, 5);
      // L_ij = A_ij Linv_j^T: Xs[q][r] = A_ij(r, q), Ys[q][c] = Linv_j(c, q)
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = wm + a * 8 + (lane >> 2), c = wn + b * 8 + 2 * (lane & 3) + h;
            Xs[0][c][r] = acc[a][b][h];
            acc[a][b][h] = 0.0;
          }
      __syncthreads();
      const double* lj = linv + static_cast<size_t>(j) * 1024;
      for (int e = t; e < 1024; e += 128) Ys[0][e >> 5][e & 31] = __ldcg(lj + e);
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < 32; kk += 4) {
        double a[2], b[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) a[q] = Xs[0][kk + (lane & 3)][wm + q * 8 + (lane >> 2)];
#pragma unroll
        for (int q = 0; q < 2; ++q) b[q] = Ys[0][kk + (lane & 3)][wn + q * 8 + (lane >> 2)];
#pragma unroll
        for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
          for (int b2 = 0; b2 < 2; ++b2) dmma(acc[a2][b2][0], acc[a2][b2][1], a[a2], b[b2]);
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = wm + a * 8 + (lane >> 2), c = wn + b * 8 + 2 * (lane & 3) + h;
            if (r < ib && c < jb) A[(i0 + r) + static_cast<size_t>(j0 + c) * lda] = acc[a][b][h];
          }
    }
    __syncthreads();
    if (t == 0) st_release(fl(i, j), epoch);
    if (i == j + 1) TLG_TR(j, 6);
  }
}

#ifdef TLG_FLOW_TRACE
extern "C" int tlg_debug_flow_trace(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, tlg_flow_trace, sizeof(tlg_flow_trace)) != cudaSuccess) return 1;
  return cudaMemcpyFromSymbol(out + kTrN * 8, tlg_flow_trace2, sizeof(tlg_flow_trace2)) == cudaSuccess ? 0 : 1;
}
#endif

void potrf_lower32(tlg_ctx* ctx, double* A, int n, int lda, int* info, double* X, int ldx,
                   int band) {
  const int nt = (n + NB32 - 1) / NB32;
  int bwt = std::min(nt - 1, (std::max(band, 0) + NB32 - 1) / NB32);
  double* linv = ctx->ws<double>(S_LINV, static_cast<size_t>(nt) * NB32 * NB32);
  ctx->linv_owner = nullptr;  // 32-wide inverse tiles: not usable by trsm_left_lower
  ctx->linv32_owner = A;
  if (!ctx->force_coop_potrf) {
    // the task dataflow (k_potrf_flow32); with X, the L^-1 tiles as further
    // tasks (the strictly upper tiles of X are zeroed here)
    const size_t nflag = static_cast<size_t>(nt) * (bwt + 1) + (X ? static_cast<size_t>(nt) * nt : 0);
    int* flags = ctx->ws<int>(S_FLOWFLAG, nflag + 4);
    unsigned long long* counter = reinterpret_cast<unsigned long long*>(flags + nflag + (nflag & 1));
    TLG_CUDA(cudaMemsetAsync(flags, 0, (nflag + 4) * sizeof(int), ctx->stream));
    if (X) TLG_CUDA(cudaMemset2DAsync(X, sizeof(double) * ldx, 0, sizeof(double) * n, n, ctx->stream));
    int per_sm = 0;
    TLG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_potrf_flow32, 128, 0));
    long long tasks = static_cast<long long>(nt - bwt) * (bwt + 1) + static_cast<long long>(bwt) * (bwt + 1) / 2;
    if (X) tasks += static_cast<long long>(nt) * (nt + 1) / 2;
    const int grid = static_cast<int>(std::max<long long>(1, std::min<long long>(tasks, static_cast<long long>(ctx->num_sms) * std::max(1, std::min(per_sm, TLG_PF_MINB)))));
    int epoch = 1;
    // Factor-task claim order: by key j S + (i - j), ties by ascending j.
    // S = 2 (default) is the anti-diagonal order i + j, the wavefront of the
    // tile dependencies: every dependency of a task has a smaller key for any
    // S >= 2, so every wait still targets an earlier-claimed task (deadlock-
    // free with co-resident CTAs); near-diagonal tasks of the next columns are
    // claimed before the far rows of the current one (C5: 51 -> 42 ms against
    // column-major, S = bwt + 1; env TLG_POTRF_SKEW overrides, 1 = column-major).
    const int2* order = nullptr;
    const char* sk = std::getenv("TLG_POTRF_SKEW");
    const int skew = sk ? std::atoi(sk) : 2;
    if (skew >= 2 && skew <= std::max(bwt, 2)) {
      // L^-1 tasks (with X) join the same order: row i's X tiles get the key
      // just above row i's last factor task (diagonal key i S), ascending j;
      // their dependencies (L_ik, Linv_i, X_kj for k < i) all have smaller keys
      const size_t nfac = static_cast<size_t>(nt - bwt) * (bwt + 1) + static_cast<size_t>(bwt) * (bwt + 1) / 2;
      const size_t ntask = nfac + (X ? static_cast<size_t>(nt) * (nt + 1) / 2 : 0);
      int2* dorder = ctx->ws<int2>(S_FLOWORDER, ntask);
      const long long key = (static_cast<long long>(nt) << 32) ^ (static_cast<long long>(bwt) << 12) ^
                            (skew << 1) ^ (X ? 1 : 0);
      if (ctx->flow_order_key != key) {
        std::vector<int2>& host = ctx->flow_order_host;
        host.clear();
        host.reserve(ntask);
        const long long kmax = static_cast<long long>(nt - 1) * skew + bwt;
        for (long long K = 0; K <= kmax; ++K) {
          const long long jlo = std::max<long long>(0, (K - bwt + skew - 1) / skew);
          const long long jhi = std::min<long long>(nt - 1, K / skew);
          for (long long jj = jlo; jj <= jhi; ++jj) {
            const long long ii = jj + (K - jj * skew);
            if (ii < nt) host.push_back(make_int2(static_cast<int>(ii), static_cast<int>(jj)));
          }
          // X row i after its diagonal task (key i S)
          if (X && K % skew == 0 && K / skew < nt) {
            const int ii = static_cast<int>(K / skew);
            for (int jj = 0; jj <= ii; ++jj) host.push_back(make_int2(ii, -1 - jj));
          }
        }
        require(host.size() == ntask, TLG_RUNTIME_ERROR, "potrf: task order size");
        TLG_CUDA(cudaMemcpyAsync(dorder, host.data(), host.size() * sizeof(int2), cudaMemcpyHostToDevice,
                                 ctx->stream));
        ctx->flow_order_key = key;
      }
      order = dorder;
    }
    void* args[] = {&A, &n, &lda, &bwt, &linv, &info, &X, &ldx, &flags, &counter, &epoch, &order};
    TLG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_potrf_flow32), dim3(grid),
                                         dim3(128), args, 0, ctx->stream));
    ++ctx->launches;
    return;
  }
  int per_sm = 0;
  TLG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_potrf_coop32, 128, 0));
  int maxtiles = nt;
  for (int k = 0; k < nt; ++k) {
    const int nr = std::min(nt - 1, k + bwt) - k;
    maxtiles = std::max(maxtiles, nr * (nr + 1) / 2 + (X ? nr * (k + 1) : 0));
  }
  const int grid = std::max(1, std::min(maxtiles, ctx->num_sms * std::max(per_sm, 1)));
  void* args[] = {&A, &n, &lda, &linv, &info, &X, &ldx, &bwt};
  TLG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_potrf_coop32), dim3(grid),
                                       dim3(128), args, 0, ctx->stream));
  ++ctx->launches;
}

void potrf_lower(tlg_ctx* ctx, double* A, int n, int lda, int* info, double* X, int ldx,
                 int band) {
  if (n <= 0) return;
  if (band < 0 || band > n) band = n;
  if ((n <= kSmallN || band < n) && !ctx->force_nb64) {
    potrf_lower32(ctx, A, n, lda, info, X, ldx, band);
    return;
  }
  const int nt = (n + NB - 1) / NB;
  double* linv = ctx->ws<double>(S_LINV, static_cast<size_t>(nt) * NB * NB);
  ctx->linv_owner = A;
  ctx->linv32_owner = nullptr;
  const size_t smem = sizeof(double) * kDiagSmemDoubles;
  static bool attr = false;
  if (!attr) {
    TLG_CUDA(cudaFuncSetAttribute(k_potrf_coop, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    attr = true;
  }
  int per_sm = 0;
  TLG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_potrf_coop, 128, smem));
  int maxtiles = std::max(nt - 1, (nt - 1) * nt / 2);
  if (X) {
    for (int k = 0; k < nt; ++k)
      maxtiles = std::max(maxtiles, (nt - k - 1) * (nt - k) / 2 + (nt - k - 1) * (k + 1));
    maxtiles = std::max(maxtiles, nt);
  }
  const int grid = std::max(1, std::min(maxtiles, ctx->num_sms * std::max(per_sm, 1)));
  void* args[] = {&A, &n, &lda, &linv, &info, &X, &ldx};
  TLG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_potrf_coop), dim3(grid),
                                       dim3(128), args, smem, ctx->stream));
  ++ctx->launches;
}

void trsm_left_lower(tlg_ctx* ctx, const double* L, int n, int ldl, double* B, int nrhs,
                     int ldb, int trans) {
  if (n <= 0 || nrhs <= 0) return;
  require(ctx->linv_owner == L, TLG_RUNTIME_ERROR, "trsm: matrix was not factored last");
  const double* linv = ctx->ws<double>(S_LINV, 1);
  k_trsm_tiles<<<(nrhs + NB - 1) / NB, 128, 0, ctx->stream>>>(L, n, ldl, linv, B, nrhs, ldb, trans);
  TLG_LAUNCHED(ctx);
}

__global__ void k_symmetrize(double* __restrict__ A, int n, int lda) {
  const long long tot = (long long)n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(e % n), c = static_cast<int>(e / n);
    if (r > c) {
      const double v = 0.5 * (A[r + (size_t)c * lda] + A[c + (size_t)r * lda]);
      A[r + (size_t)c * lda] = v;
      A[c + (size_t)r * lda] = v;
    }
  }
}

void symmetrize(tlg_ctx* ctx, double* A, int n, int lda) {
  if (n <= 1) return;
  const long long tot = (long long)n * n;
  const unsigned b = static_cast<unsigned>(std::min<long long>((tot + 255) / 256, 4ull * ctx->num_sms));
  k_symmetrize<<<b, 256, 0, ctx->stream>>>(A, n, lda);
  TLG_LAUNCHED(ctx);
}

__global__ void k_add_diag(double* __restrict__ A, int n, int lda, double v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) A[i + (size_t)i * lda] += v;
}

void add_diag(tlg_ctx* ctx, double* A, int n, int lda, double v) {
  if (n <= 0) return;
  k_add_diag<<<(n + 255) / 256, 256, 0, ctx->stream>>>(A, n, lda, v);
  TLG_LAUNCHED(ctx);
}

}  // namespace tlg
