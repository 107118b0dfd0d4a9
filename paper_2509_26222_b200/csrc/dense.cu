// Dense FP64 kernels for the kernel-matrix update: a DMMA (mma.sync
// m8n8k4 f64, the sm_100a FP64 tensor path — tcgen05 has no f64 kind) GEMM
// with 64x64 CTA tiles; a tile Cholesky in ONE cooperative launch (per 64-wide
// step: the diagonal tile is factored and inverted in shared memory by one
// CTA, panel tiles become GEMMs with that inverse, trailing tiles are DMMA
// GEMMs, grid barriers between the phases); and a one-launch tile TRSM where
// each CTA walks the tile rows of its 64-column slab with GEMMs only.
#include <cooperative_groups.h>

#include "dense.cuh"

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
    const int i = t & 63, h = t >> 6;
    double s0 = 0.0, s1 = 0.0;
    if (i < mb) {
      const double* a = d.A + m0 + i;
      int k = h;
      for (; k + 2 < K; k += 4) {
        s0 = fma(a[(size_t)k * d.lda], bval(k), s0);
        s1 = fma(a[(size_t)(k + 2) * d.lda], bval(k + 2), s1);
      }
      for (; k < K; k += 2) s0 = fma(a[(size_t)k * d.lda], bval(k), s0);
    }
    red[t] = s0 + s1;
  } else {
    const int lane = t & 31, w = t >> 5;
    for (int i = w; i < mb; i += 4) {
      const double* a = d.A + (size_t)(m0 + i) * d.lda;
      double s = 0.0;
      for (int k = lane; k < K; k += 32) s = fma(a[k], bval(k), s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) red[i] = s;
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

void gemm(tlg_ctx* ctx, const GemmDesc& d) {
  if (d.M <= 0 || d.N <= 0) return;
  dim3 grid((d.M + TM - 1) / TM, (d.N + TN - 1) / TN);
  k_gemm<<<grid, 128, 0, ctx->stream>>>(d);
  TLG_LAUNCHED(ctx);
}

void gemm_grouped(tlg_ctx* ctx, const GemmDesc* d_descs, int count, int max_m, int max_n) {
  if (count <= 0 || max_m <= 0 || max_n <= 0) return;
  dim3 grid((max_m + TM - 1) / TM, (max_n + TN - 1) / TN, count);
  k_gemm_grouped<<<grid, 128, 0, ctx->stream>>>(d_descs);
  TLG_LAUNCHED(ctx);
}


// ---------------------------------------------------------------------------
// Tile factorisation. NB = 64-wide tiles; every tile step is one CTA of 128
// threads running gemm_tile (DMMA) or the diagonal-tile routine below.
constexpr int NB = 64;

// Cholesky of the kb x kb diagonal tile (lower) in shared memory, written
// back to A, plus the inverse of the factor, Linv (64 x 64, ld 64, zero
// above the diagonal), so off-diagonal triangular solves become DMMA GEMMs.
// `a` is dynamic shared memory of NB x (NB + 1) doubles.
// Register-blocked version (128 threads): thread t owns the 4 x 8 block
// rows 4*(t>>3).., cols 8*(t&7).. of both L and X = L^-1. Step j factors
// column j (pivot, scale) and eliminates row j of the identity in the same
// pass; the only shared traffic is column j of L and row j of X (double
// buffered), two barriers per step.
__device__ void tile_potrf_inv_reg(double* __restrict__ A, int lda, int kb,
                                   double* __restrict__ linv, int* __restrict__ info,
                                   double* sh) {
  const int t = threadIdx.x;
  const int r0 = (t >> 3) * 4, c0 = (t & 7) * 8;
  double* colL = sh;        // [2][64]
  double* rowX = sh + 128;  // [2][64]
  double* piv = sh + 256;   // [2]
  double a[4][8], x[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = r0 + i, c = c0 + k;
      a[i][k] = (r < kb && c < kb) ? (r >= c ? A[r + (size_t)c * lda] : 0.0) : (r == c ? 1.0 : 0.0);
      x[i][k] = (r == c) ? 1.0 : 0.0;
    }
  for (int j = 0; j < NB; ++j) {
    const int buf = (j & 1) * 64;
    // 1. pivot (owner of (j, j))
    if (j >= r0 && j < r0 + 4 && j >= c0 && j < c0 + 8) {
      double d = 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (r0 + i == j && c0 + k == j) d = a[i][k];
      if (!(d > 0.0) || !isfinite(d)) atomicOr(info, 1);
      const double l = sqrt(d);
      piv[(j & 1)] = l;
    }
    __syncthreads();
    const double l = piv[j & 1];
    const double il = 1.0 / l;
    // 2. column j of L (rows > j scaled) and row j of X (scaled)
    if (j >= c0 && j < c0 + 8) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = r0 + i;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (c0 + k == j) {
            if (r > j) a[i][k] *= il;
            else if (r == j) a[i][k] = l;
            colL[buf + r] = (r >= j) ? a[i][k] : 0.0;
          }
      }
    }
    if (j >= r0 && j < r0 + 4) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (r0 + i == j) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            x[i][k] *= il;
            rowX[buf + c0 + k] = x[i][k];
          }
        }
    }
    __syncthreads();
    // 3. trailing update of L and elimination of X
    double cr[4], cc[8], rx[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) cr[i] = colL[buf + r0 + i];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      cc[k] = colL[buf + c0 + k];
      rx[k] = rowX[buf + c0 + k];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = r0 + i;
      if (r > j) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int c = c0 + k;
          if (c > j && c <= r) a[i][k] = fma(-cr[i], cc[k], a[i][k]);
          x[i][k] = fma(-cr[i], rx[k], x[i][k]);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = r0 + i, c = c0 + k;
      if (r < kb && c < kb && r >= c) A[r + (size_t)c * lda] = a[i][k];
      linv[r + (size_t)c * NB] = x[i][k];
    }
  __syncthreads();
}

// Branch-free register-blocked factor + inverse (128 threads, 4 x 8 blocks of
// L and X = L^-1 per thread), ONE barrier per step: the owners of column j of
// A and row j of X publish them unscaled; every thread derives the pivot
// l = sqrt(a_jj) itself and applies masked rank-1 updates. Entries above
// the diagonal of A are never read and may take garbage.
__device__ void tile_potrf_inv_v3(double* __restrict__ A, int lda, int kb,
                                  double* __restrict__ linv, int* __restrict__ info,
                                  double* sh) {
  const int t = threadIdx.x;
  const int r0 = (t >> 3) * 4, c0 = (t & 7) * 8;
  double a[4][8], x[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = r0 + i, c = c0 + k;
      a[i][k] = (r < kb && c < kb) ? (r >= c ? A[r + (size_t)c * lda] : 0.0) : (r == c ? 1.0 : 0.0);
      x[i][k] = (r == c) ? 1.0 : 0.0;
    }
  bool bad = false;
#pragma unroll 1
  for (int j = 0; j < NB; ++j) {
    double* colA = sh + (j & 1) * 128;  // column j of A (rows >= j meaningful)
    double* rowX = colA + 64;           // row j of X
    const int jc = j - c0, jr = j - r0;
    if (jc >= 0 && jc < 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k == jc)
#pragma unroll
          for (int i = 0; i < 4; ++i) colA[r0 + i] = a[i][k];
    }
    if (jr >= 0 && jr < 4) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i == jr)
#pragma unroll
          for (int k = 0; k < 8; ++k) rowX[c0 + k] = x[i][k];
    }
    __syncthreads();
    const double d = colA[j];
    bad |= !(d > 0.0) || !isfinite(d);
    const double il = rsqrt(d);
    const double l = d * il;
    double cr[4], cc[8], rx[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) cr[i] = (r0 + i > j) ? colA[r0 + i] * il : 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      cc[k] = (c0 + k > j) ? colA[c0 + k] * il : 0.0;
      rx[k] = rowX[c0 + k] * il;
    }
    // column j of L and row j of X become final
    if (jc >= 0 && jc < 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k == jc)
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i][k] = (r0 + i == j) ? l : cr[i];
    }
    if (jr >= 0 && jr < 4) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i == jr)
#pragma unroll
          for (int k = 0; k < 8; ++k) x[i][k] = rx[k];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        a[i][k] = fma(-cr[i], cc[k], a[i][k]);
        x[i][k] = fma(-cr[i], rx[k], x[i][k]);
      }
  }
  if (bad && t == 0) atomicOr(info, 1);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = r0 + i, c = c0 + k;
      if (r < kb && c < kb && r >= c) A[r + (size_t)c * lda] = a[i][k];
      linv[r + (size_t)c * NB] = x[i][k];
    }
  __syncthreads();
}

// Compact diagonal-tile factor + inverse in shared memory with rolled loops
// (straight-line unrolled code of this size is instruction-cache bound).
// LDL^T-style elimination: pivot j subtracts a_rj a_cj / d_j from the
// trailing lower block and eliminates row j of the unit inverse; one barrier
// per pivot; square roots are applied at the end:
//   L = L_unit D^(1/2) -> L_rc = a_rc / sqrt(d_c),  L^-1 = D^(-1/2) X_unit.
// Thread t: rows {p, 63 - p} (p = t & 31, balances work), columns = t>>5 mod 4.
// sh: 2 * 64 * 65 + 64 doubles.
__device__ void tile_potrf_inv_s(double* __restrict__ A, int lda, int kb,
                                 double* __restrict__ linv, int* __restrict__ info, double* sh) {
  const int t = threadIdx.x;
  double(*a)[65] = reinterpret_cast<double(*)[65]>(sh);
  double(*x)[65] = reinterpret_cast<double(*)[65]>(sh + 64 * 65);
  double* isd = sh + 2 * 64 * 65;
  // pivot column of A and pivot row of X, double buffered in arrays that the
  // update loops never write, so their loads overlap across iterations
  double(*colb)[64] = reinterpret_cast<double(*)[64]>(sh + 2 * 64 * 65 + 64);
  double(*rowb)[64] = reinterpret_cast<double(*)[64]>(sh + 2 * 64 * 65 + 192);
  for (int e = t; e < 64 * 64; e += blockDim.x) {
    const int r = e & 63, c = e >> 6;
    const double v = (r < kb && c < kb) ? (r >= c ? A[r + (size_t)c * lda] : 0.0) : (r == c ? 1.0 : 0.0);
    a[r][c] = v;
    x[r][c] = (r == c) ? 1.0 : 0.0;
    if (c == 0) colb[0][r] = v;
    if (r == 0) rowb[0][c] = (c == 0) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int p = t & 31, cp = t >> 5;
  bool bad = false;
#pragma unroll 1
  for (int j = 0; j < NB; ++j) {
    const double* col = colb[j & 1];
    const double* xr = rowb[j & 1];
    double* coln = colb[(j + 1) & 1];
    double* xrn = rowb[(j + 1) & 1];
    const double d = col[j];
    bad |= !(d > 0.0) || !isfinite(d);
    const double is = rsqrt(d);
    const double dinv = is * is;
    if (t == 0) isd[j] = is;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = h ? 63 - p : p;
      if (r > j) {
        const double f = col[r] * dinv;
        const int cs = j + 1 + ((cp - j - 1) & 3);
#pragma unroll 4
        for (int c = cs; c <= r; c += 4) {
          const double v = fma(-f, col[c], a[r][c]);
          a[r][c] = v;
          if (c == j + 1) coln[r] = v;  // next pivot column
        }
#pragma unroll 4
        for (int c = cp; c <= j; c += 4) {
          const double v = fma(-f, xr[c], x[r][c]);
          x[r][c] = v;
          if (r == j + 1) xrn[c] = v;  // next pivot row of X
        }
        if (r == j + 1 && cp == ((j + 1) & 3)) xrn[j + 1] = 1.0;
      }
    }
    __syncthreads();
  }
  if (bad && t == 0) atomicOr(info, 1);
  for (int e = t; e < 64 * 64; e += blockDim.x) {
    const int r = e & 63, c = e >> 6;
    if (r < kb && c < kb && r >= c) A[r + (size_t)c * lda] = a[r][c] * isd[c];
    linv[r + (size_t)c * NB] = (r >= c) ? x[r][c] * isd[r] : 0.0;
  }
  __syncthreads();
}

// Warp-synchronous 32 x 32 Cholesky + inverse: lane i owns row i of A and
// of X = L^-1 in registers; per pivot the column of L and the row of X are
// broadcast through shared memory with __syncwarp only (no block barrier).
// In: S (ld 33) lower part. Out: L (lower, zeros above) and X into S / Xs.
__device__ __forceinline__ void warp_potrf_inv32(double* S, double* Xs, double* bc, bool& bad) {
  const int i = threadIdx.x & 31;
  double a[32], x[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    a[c] = (c <= i) ? S[i * 33 + c] : 0.0;
    x[c] = (c == i) ? 1.0 : 0.0;
  }
  double* colL = bc;       // [32]
  double* rowX = bc + 32;  // [32]
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    // pivot row j publishes its diagonal and its X row
    if (i == j) {
      colL[j] = a[j];
#pragma unroll
      for (int c = 0; c < 32; ++c) rowX[c] = x[c];
    }
    __syncwarp();
    const double d = colL[j];
    bad |= !(d > 0.0) || !isfinite(d);
    const double il = rsqrt(d);
    const double lij = (i > j) ? a[j] * il : (i == j ? d * il : 0.0);
    a[j] = lij;
    __syncwarp();
    colL[i] = lij;  // column j of L (zero above the pivot)
    __syncwarp();
    if (i == j) {
#pragma unroll
      for (int c = 0; c <= j; ++c) x[c] *= il;
    } else if (i > j) {
#pragma unroll
      for (int c = 0; c <= j; ++c) x[c] = fma(-lij, rowX[c] * il, x[c]);
    }
#pragma unroll
    for (int c = j + 1; c < 32; ++c) a[c] = fma(-lij, colL[c], a[c]);
    __syncwarp();
  }
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    S[i * 33 + c] = (c <= i) ? a[c] : 0.0;
    Xs[i * 33 + c] = x[c];
  }
  __syncwarp();
}

// 64 x 64 diagonal tile from two warp-level 32 blocks (128 threads):
//   L11 = chol(A11), X11 = L11^-1;  L21 = A21 X11^T;  A22 -= L21 L21^T;
//   L22 = chol(A22), X22 = L22^-1;  X21 = -X22 L21 X11.
// sh: >= 4 * 32 * 33 + 64 doubles.
__device__ void tile_potrf_inv_w32(double* __restrict__ A, int lda, int kb,
                                   double* __restrict__ linv, int* __restrict__ info,
                                   double* sh) {
  const int t = threadIdx.x, w = t >> 5;
  double* B11 = sh;                // row-major [32][33]: A11 -> L11
  double* B21 = sh + 32 * 33;      // A21 -> L21
  double* B22 = sh + 2 * 32 * 33;  // A22 -> L22
  double* X = sh + 3 * 32 * 33;    // X11, then X22
  double* bc = sh + 4 * 32 * 33;   // 64 doubles broadcast area
  for (int e = t; e < 64 * 64; e += blockDim.x) {
    const int r = e & 63, c = e >> 6;
    double v = (r < kb && c < kb) ? A[r + (size_t)c * lda] : (r == c ? 1.0 : 0.0);
    if (r < 32 && c < 32) B11[r * 33 + c] = v;
    else if (r >= 32 && c < 32) B21[(r - 32) * 33 + c] = v;
    else if (r >= 32 && c >= 32) B22[(r - 32) * 33 + (c - 32)] = v;
  }
  __syncthreads();
  bool bad = false;
  if (w == 0) warp_potrf_inv32(B11, X, bc, bad);
  __syncthreads();
  // L21 = A21 X11^T : thread owns row r = t >> 2, 8 columns (t & 3) * 8
  {
    const int r = t >> 2, cbase = (t & 3) * 8;
    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    for (int k = 0; k < 32; ++k) {
      const double av = B21[r * 33 + k];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = fma(av, X[(cbase + q) * 33 + k], acc[q]);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 8; ++q) B21[r * 33 + cbase + q] = acc[q];
    __syncthreads();
    // A22 -= L21 L21^T (lower part used)
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    for (int k = 0; k < 32; ++k) {
      const double lv = B21[r * 33 + k];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = fma(lv, B21[(cbase + q) * 33 + k], acc[q]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) B22[r * 33 + cbase + q] -= acc[q];
  }
  __syncthreads();
  // keep X11 (needed for X21) in registers of the same layout
  double x11[8];
  {
    const int r = t >> 2, cbase = (t & 3) * 8;
#pragma unroll
    for (int q = 0; q < 8; ++q) x11[q] = X[r * 33 + cbase + q];
  }
  __syncthreads();
  if (w == 0) warp_potrf_inv32(B22, X, bc, bad);
  __syncthreads();
  // X21 = -X22 (L21 X11): T = L21 X11 first
  {
    const int r = t >> 2, cbase = (t & 3) * 8;
    // stash X11 in B11's upper-unused? use B11 storage after writing L11 out
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int c = cbase + q;
      // write L11 (lower) to A now, then reuse B11 for X11
      if (r < kb && c < kb && r >= c) A[r + (size_t)c * lda] = B11[r * 33 + c];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 8; ++q) B11[r * 33 + cbase + q] = x11[q];
    __syncthreads();
    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    for (int k = 0; k < 32; ++k) {
      const double lv = B21[r * 33 + k];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = fma(lv, B11[k * 33 + cbase + q], acc[q]);
    }
    // write L21, L22 to A before overwriting B21 with T
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int c = cbase + q;
      if (32 + r < kb && c < kb) A[(32 + r) + (size_t)c * lda] = B21[r * 33 + c];
      if (32 + r < kb && 32 + c < kb && r >= c)
        A[(32 + r) + (size_t)(32 + c) * lda] = B22[r * 33 + c];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 8; ++q) B21[r * 33 + cbase + q] = acc[q];  // T
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    for (int k = 0; k < 32; ++k) {
      const double xv = X[r * 33 + k];  // X22[r][k]
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = fma(xv, B21[k * 33 + cbase + q], acc[q]);
    }
    // Linv (64 x 64, ld 64): [X11 0; X21 X22]
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int c = cbase + q;
      linv[r + (size_t)c * NB] = x11[q];
      linv[r + (size_t)(32 + c) * NB] = 0.0;
      linv[(32 + r) + (size_t)c * NB] = -acc[q];
      linv[(32 + r) + (size_t)(32 + c) * NB] = X[r * 33 + c];
    }
  }
  if (bad) atomicOr(info, 1);
  __syncthreads();
}

// 4-column blocked version (128 threads, 4 x 8 register blocks of L and
// X = L^-1): 16 steps. Step j = 4s: the owners of columns j..j+3 of A and of
// rows j..j+3 of X publish them; owners factor the 4x4 diagonal block (and
// invert it) in registers, publish the final L columns and X rows; every
// thread applies the rank-4 update. Two barriers per step.
__device__ void tile_potrf_inv_b4(double* __restrict__ A, int lda, int kb,
                                  double* __restrict__ linv, int* __restrict__ info,
                                  double* sh) {
  const int t = threadIdx.x;
  const int r0 = (t >> 3) * 4, c0 = (t & 7) * 8;
  double* rawA = sh;        // [4][64]  columns j..j+3 of A
  double* rawX = sh + 256;  // [4][64]  rows j..j+3 of X
  double* finL = sh + 512;  // [4][64]  final L columns j..j+3 (0 above the block)
  double* finX = sh + 768;  // [4][64]  final X rows j..j+3
  double a[4][8], x[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = r0 + i, c = c0 + k;
      a[i][k] = (r < kb && c < kb) ? (r >= c ? A[r + (size_t)c * lda] : 0.0) : (r == c ? 1.0 : 0.0);
      x[i][k] = (r == c) ? 1.0 : 0.0;
    }
  bool bad = false;
#pragma unroll 1
  for (int j = 0; j < NB; j += 4) {
    const bool colown = c0 == (j & ~7);
    const bool hi = (j & 4) != 0;  // columns j..j+3 are the upper half of the 8-column group
    const bool rowown = r0 == j;
    if (colown) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int i = 0; i < 4; ++i) rawA[q * 64 + r0 + i] = hi ? a[i][4 + q] : a[i][q];
    }
    if (rowown) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int k = 0; k < 8; ++k) rawX[q * 64 + c0 + k] = x[q][k];
    }
    TLG_PHASE(0);
    __syncthreads();
    TLG_PHASE(1);
    if (colown || rowown) {
      // 4x4 Cholesky of D (rows/cols j..j+3) and the inverse of its factor
      double D[4][4];
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q <= p; ++q) D[p][q] = rawA[q * 64 + j + p];
      double L[4][4], Li[4][4], iv[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        double d = D[p][p];
#pragma unroll
        for (int k = 0; k < p; ++k) d = fma(-L[p][k], L[p][k], d);
        bad |= !(d > 0.0) || !isfinite(d);
        iv[p] = rsqrt(d);
        L[p][p] = d * iv[p];
#pragma unroll
        for (int r = p + 1; r < 4; ++r) {
          double s = D[r][p];
#pragma unroll
          for (int k = 0; k < p; ++k) s = fma(-L[r][k], L[p][k], s);
          L[r][p] = s * iv[p];
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        Li[c][c] = iv[c];
#pragma unroll
        for (int r = c + 1; r < 4; ++r) {
          double s = 0.0;
#pragma unroll
          for (int k = c; k < r; ++k) s = fma(L[r][k], Li[k][c], s);
          Li[r][c] = -iv[r] * s;
        }
      }
      if (colown) {
        // L_r[q] = sum_p a_r[p] Li[q][p] for rows below the block
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = r0 + i;
          double ar[4];
#pragma unroll
          for (int p = 0; p < 4; ++p) ar[p] = rawA[p * 64 + r];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            double v;
            if (r > j + 3) {
              v = 0.0;
#pragma unroll
              for (int p = 0; p <= q; ++p) v = fma(ar[p], Li[q][p], v);
            } else if (r >= j) {
              const int pr = r - j;
              v = 0.0;
#pragma unroll
              for (int p = 0; p < 4; ++p)
                if (p == pr && q <= p) v = L[p][q];
            } else {
              v = 0.0;
            }
            finL[q * 64 + r] = v;
            if (r >= j) {
              if (hi) a[i][4 + q] = v;
              else a[i][q] = v;
            }
          }
        }
      }
      if (rowown) {
        // X rows j..j+3 final: Xf[q][c] = sum_p Li[q][p] rawX[p][c]
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          double xr[4];
#pragma unroll
          for (int p = 0; p < 4; ++p) xr[p] = rawX[p * 64 + c0 + k];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            double v = 0.0;
#pragma unroll
            for (int p = 0; p <= q; ++p) v = fma(Li[q][p], xr[p], v);
            finX[q * 64 + c0 + k] = v;
            x[q][k] = v;
          }
        }
      }
    }
    TLG_PHASE(2);
    __syncthreads();
    TLG_PHASE(3);
    // rank-4 update: A -= L_J L_J^T (columns > j+3), X -= L_J X_J (rows > j+3)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double cr[4], cc[8], rx[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) cr[i] = (r0 + i > j + 3) ? finL[q * 64 + r0 + i] : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        cc[k] = (c0 + k > j + 3) ? finL[q * 64 + c0 + k] : 0.0;
        rx[k] = finX[q * 64 + c0 + k];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          a[i][k] = fma(-cr[i], cc[k], a[i][k]);
          x[i][k] = fma(-cr[i], rx[k], x[i][k]);
        }
    }
  }
  TLG_PHASE(4);
  if (bad) atomicOr(info, 1);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = r0 + i, c = c0 + k;
      if (r < kb && c < kb && r >= c) A[r + (size_t)c * lda] = a[i][k];
      linv[r + (size_t)c * NB] = x[i][k];
    }
  __syncthreads();
}

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

__device__ void tile_potrf_inv(double* __restrict__ A, int lda, int kb, double* __restrict__ linv,
                               int* __restrict__ info, double (*a)[NB + 1], double* dinv) {
  const int t = threadIdx.x;
  for (int e = t; e < NB * NB; e += blockDim.x) {
    const int r = e % NB, c = e / NB;
    a[r][c] = (r < kb && c < kb && r >= c) ? A[r + (size_t)c * lda] : (r == c ? 1.0 : 0.0);
  }
  __syncthreads();
  for (int j = 0; j < kb; ++j) {
    const double d = a[j][j];
    const bool ok = d > 0.0 && isfinite(d);
    const double l = sqrt(d);
    const double inv = 1.0 / l;
    __syncthreads();
    if (t == 0) {
      if (!ok) atomicOr(info, 1);
      a[j][j] = l;
      dinv[j] = inv;
    }
    for (int i = j + 1 + t; i < kb; i += blockDim.x) a[i][j] *= inv;
    __syncthreads();
    const int rem = kb - j - 1;
    for (int e = t; e < rem * rem; e += blockDim.x) {
      const int r = j + 1 + e % rem, c = j + 1 + e / rem;
      if (r >= c) a[r][c] = fma(-a[r][j], a[c][j], a[r][c]);
    }
    __syncthreads();
  }
  for (int i = kb + t; i < NB; i += blockDim.x) dinv[i] = 1.0;  // identity padding
  for (int e = t; e < kb * kb; e += blockDim.x) {
    const int r = e % kb, c = e / kb;
    if (r >= c) A[r + (size_t)c * lda] = a[r][c];
  }
  __syncthreads();
  // Inverse by row sweep, columns in parallel: thread pair (2c, 2c+1) owns
  // column c; thread h keeps x[k][c] for k = h (mod 2) in registers, partial
  // dot products combine with one shuffle. No block barriers needed.
  const int c = t >> 1, h = t & 1;
  double xr[NB / 2];
#pragma unroll
  for (int q = 0; q < NB / 2; ++q) xr[q] = 0.0;
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    double p0 = 0.0, p1 = 0.0;
#pragma unroll
    for (int q = 0; q < NB / 2; ++q) {
      if (2 * q + 1 < i) {
        if (q & 1) p1 = fma(a[i][2 * q + h], xr[q], p1);
        else p0 = fma(a[i][2 * q + h], xr[q], p0);
      } else if (2 * q < i) {  // k = 2q + h < i only for h = 0
        if (h == 0) p0 = fma(a[i][2 * q], xr[q], p0);
      }
    }
    double p = p0 + p1;
    p += __shfl_xor_sync(0xffffffffu, p, 1);
    const double xi = (i == c) ? dinv[i] : (i > c ? -p * dinv[i] : 0.0);
    if ((i & 1) == h) xr[i >> 1] = xi;
  }
  if (c < NB) {
#pragma unroll
    for (int q = 0; q < NB / 2; ++q) linv[(2 * q + h) + (size_t)c * NB] = xr[q];
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

// One warp: L L^T = A for the kb x kb (kb <= 32) lower tile at A (lda), padded
// with the identity; writes L back into A and X = L^-1 (32 x 32, ld 32,
// zero above the diagonal) into linv. sh: kWarpPotrfSmem doubles.
constexpr int kWarpPotrfSmem = 2 * 32 + 32 * 33 + 32;
__device__ void warp_potrf_inv32(double* __restrict__ A, int lda, int kb,
                                 double* __restrict__ linv, int* __restrict__ info,
                                 double* __restrict__ sh) {
  const int i = threadIdx.x & 31;
  double* col = sh;            // [2][32] broadcast of the current column of L
  double* xs = sh + 64;        // [32][33] transpose buffer
  double* dinv = xs + 32 * 33;  // [32] 1 / L_jj
  double a[32];
#pragma unroll
  for (int k = 0; k < 32; ++k)
    a[k] = (i < kb && k < kb) ? (k <= i ? A[i + (size_t)k * lda] : 0.0) : (i == k ? 1.0 : 0.0);
  TLG_PHASE(1);
  bool bad = false;
  double d = __shfl_sync(0xffffffffu, a[0], 0);
  // Right-looking, lane i = row i. Entries above the diagonal hold garbage
  // that is never read (pivots and columns only read k <= i).
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    bad |= !(d > 0.0) || !isfinite(d);
    const double rs = rsqrt(d);
    const double l = (i == j) ? d * rs : a[j] * rs;
    a[j] = l;
    if (i == j) dinv[j] = rs;
    if (j + 1 < 32) {
      // next pivot straight from the owner's own value (l_{j+1,j} = its l)
      const double dn = fma(-l, l, a[j + 1]);
      double* cb = col + (j & 1) * 32;
      cb[i] = l;
      d = __shfl_sync(0xffffffffu, dn, j + 1);
      __syncwarp();
#pragma unroll
      for (int p = 0; p < 16; ++p) {
        if (2 * p + 1 <= j) continue;  // both columns already eliminated
        const double2 v = *reinterpret_cast<const double2*>(cb + 2 * p);
        if (2 * p > j) a[2 * p] = fma(-l, v.x, a[2 * p]);
        a[2 * p + 1] = fma(-l, v.y, a[2 * p + 1]);
      }
    }
  }
  TLG_PHASE(2);
  if (bad && i == 0) atomicOr(info, 1);
  // L back to A (lower part only) and to the transpose buffer (row i)
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (k <= i && i < kb && k < kb) A[i + (size_t)k * lda] = a[k];
    xs[i * 33 + k] = (k <= i) ? a[k] : 0.0;
  }
  __syncwarp();
  // X = L^-1, lane c = column c: X[k][c] = (delta_kc - sum_{p<k} L[k][p] X[p][c]) / L[k][k]
  // accumulated right-looking so each row is one fma + one mul after the last.
  TLG_PHASE(3);
  double x[32];  // running right-hand side, becomes X[:, i] in place
#pragma unroll
  for (int k = 0; k < 32; ++k) x[k] = (k == i) ? 1.0 : 0.0;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    x[k] *= dinv[k];
#pragma unroll
    for (int r = k + 1; r < 32; ++r) x[r] = fma(-xs[r * 33 + k], x[k], x[r]);
  }
  TLG_PHASE(4);
  __syncwarp();
  // transpose so that the store of linv (column-major) is coalesced
#pragma unroll
  for (int k = 0; k < 32; ++k) xs[k * 33 + i] = x[k];
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 32; ++c) linv[i + (size_t)c * NB32] = xs[i * 33 + c];
  TLG_PHASE(5);
}

// bwt: lower tile bandwidth (tile (i, j) is zero for i - j > bwt; fill-in of
// a banded matrix stays inside the band), nt - 1 for a dense matrix.
// Lookahead schedule (two grid barriers per step): the diagonal tile k+1 is
// updated and factored by block 0 inside the trailing phase of step k, while
// the other blocks apply the rest of step k's trailing update (and X's).
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
// diagonal-tile inverses in linv), one cooperative launch, right-looking and
// one grid barrier per tile step. Forward: every CTA forms y_k = Linv_kk b_k
// (32 x 32, redundantly), then subtracts L_ik y_k from the band rows below
// (thread per row, coalesced along the row index). Backward: x_k =
// Linv_kk^T z_k, then z_c -= sum_r L_rc x_r for the band columns to the left
// (thread per column, contiguous 32-row reads).
__global__ void __launch_bounds__(128) k_band_solve_coop(const double* __restrict__ L, int n,
                                                         int ld, int bwt,
                                                         const double* __restrict__ linv,
                                                         double* __restrict__ b,
                                                         double* __restrict__ y) {
  __shared__ double sk[NB32], sv[NB32];
  cg::grid_group grid = cg::this_grid();
  const int nt = (n + NB32 - 1) / NB32;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  for (int k = 0; k < nt; ++k) {  // forward: y = L^-1 b
    const int k0 = k * NB32, kb = min(NB32, n - k0);
    if (threadIdx.x < NB32) sk[threadIdx.x] = threadIdx.x < kb ? b[k0 + threadIdx.x] : 0.0;
    __syncthreads();
    if (threadIdx.x < kb) {
      const double* Li = linv + (size_t)k * NB32 * NB32;
      double v = 0.0;
      for (int c = 0; c <= (int)threadIdx.x; ++c) v = fma(Li[threadIdx.x + c * NB32], sk[c], v);
      sv[threadIdx.x] = v;
      if (blockIdx.x == 0) y[k0 + threadIdx.x] = v;
    }
    __syncthreads();
    const int r0 = k0 + kb, r1 = min(n, (min(nt - 1, k + bwt) + 1) * NB32);
    for (int r = r0 + tid; r < r1; r += nth) {
      double acc = 0.0;
      for (int c = 0; c < kb; ++c) acc = fma(L[r + (size_t)(k0 + c) * ld], sv[c], acc);
      b[r] -= acc;
    }
    grid.sync();
  }
  for (int k = nt - 1; k >= 0; --k) {  // backward: x = L^-T y (in y)
    const int k0 = k * NB32, kb = min(NB32, n - k0);
    if (threadIdx.x < NB32) sk[threadIdx.x] = threadIdx.x < kb ? y[k0 + threadIdx.x] : 0.0;
    __syncthreads();
    if (threadIdx.x < kb) {
      const double* Li = linv + (size_t)k * NB32 * NB32;
      double v = 0.0;
      for (int r = threadIdx.x; r < kb; ++r) v = fma(Li[r + threadIdx.x * NB32], sk[r], v);
      sv[threadIdx.x] = v;
    }
    __syncthreads();
    grid.sync();  // every CTA has read y_k before block 0 overwrites it
    if (blockIdx.x == 0 && threadIdx.x < kb) y[k0 + threadIdx.x] = sv[threadIdx.x];
    const int c0 = max(0, k - bwt) * NB32;
    for (int c = c0 + tid; c < k0; c += nth) {
      const double* col = L + (size_t)c * ld + k0;
      double acc = 0.0;
      for (int r = 0; r < kb; ++r) acc = fma(col[r], sv[r], acc);
      y[c] -= acc;
    }
    grid.sync();
  }
}

void band_solve(tlg_ctx* ctx, const double* L, int n, int ld, int band, double* b) {
  if (n <= 0) return;
  require(ctx->linv32_owner == L, TLG_RUNTIME_ERROR, "band_solve: matrix was not factored last");
  const int nt = (n + NB32 - 1) / NB32;
  int bwt = std::min(nt - 1, (std::max(band, 0) + NB32 - 1) / NB32);
  const double* linv = ctx->ws<double>(S_LINV, 1);
  double* y = ctx->ws<double>(S_XINV2, n);
  int per_sm = 0;
  TLG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_band_solve_coop, 128, 0));
  const int rows = (bwt + 1) * NB32;
  const int grid = std::max(1, std::min((rows + 127) / 128, ctx->num_sms * std::max(per_sm, 1)));
  void* args[] = {&L, &n, &ld, &bwt, &linv, &b, &y};
  TLG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_band_solve_coop), dim3(grid),
                                       dim3(128), args, 0, ctx->stream));
  ++ctx->launches;
  TLG_CUDA(cudaMemcpyAsync(b, y, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToDevice, ctx->stream));
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

static void potrf_lower32(tlg_ctx* ctx, double* A, int n, int lda, int* info, double* X,
                          int ldx, int band) {
  const int nt = (n + NB32 - 1) / NB32;
  int bwt = std::min(nt - 1, (std::max(band, 0) + NB32 - 1) / NB32);
  double* linv = ctx->ws<double>(S_LINV, static_cast<size_t>(nt) * NB32 * NB32);
  ctx->linv_owner = nullptr;  // 32-wide inverse tiles: not usable by trsm_left_lower
  ctx->linv32_owner = A;
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
  const size_t smem = sizeof(double) * std::max(kDiagSmemDoubles, 2 * 64 * 65 + 64 + 256);
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

__global__ void __launch_bounds__(128) k_diag_tile_only(double* A, int lda, double* linv, int* info,
                                                        int reps) {
  extern __shared__ double shd[];
  for (int r = 0; r < reps; ++r) TLG_DIAG_TILE(A, lda, 64, linv, info, shd);
}

__global__ void __launch_bounds__(128) k_gridsync_only(int reps) {
  cg::grid_group grid = cg::this_grid();
  for (int r = 0; r < reps; ++r) grid.sync();
}

__global__ void k_zero_upper(double* A, int n) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * n;
       e += (long long)gridDim.x * blockDim.x)
    if (e / n > e % n) A[e] = 0.0;
}

__global__ void k_spd_fill(double* A, int n, unsigned seed) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * n;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(e % n), c = static_cast<int>(e / n);
    const int lo = min(r, c), hi = max(r, c);
    const unsigned hsh = (lo * 2654435761u) ^ (hi * 40503u) ^ seed;
    A[e] = (r == c ? n : 0.0) + ((hsh % 1000) / 1000.0 - 0.5);
  }
}

// Dense-layer microbenchmark (tlg_debug_dense_bench): op 0 = potrf, 1 = trsm
// with nrhs columns, 2 = single 64x64x64 tile GEMM per CTA over `reps` CTAs.
double dense_bench(tlg_ctx* ctx, int op, int n, int nrhs, int reps) {
  cudaStream_t s = ctx->stream;
  DBuf<double> A, B;
  A.ensure(static_cast<size_t>(n) * n);
  B.ensure(static_cast<size_t>(n) * std::max(nrhs, op == 5 ? n : 1));
  DBuf<int> info;
  info.ensure(1);
  TLG_CUDA(cudaMemsetAsync(info.p, 0, sizeof(int), s));
  cudaEvent_t e0, e1;
  TLG_CUDA(cudaEventCreate(&e0));
  TLG_CUDA(cudaEventCreate(&e1));
  float best = 1e30f;
  for (int it = 0; it < reps; ++it) {
    k_spd_fill<<<256, 256, 0, s>>>(A.p, n, 12345u + it);
    TLG_CUDA(cudaMemsetAsync(B.p, 0, sizeof(double) * n * std::max(nrhs, op == 5 ? n : 1), s));
    ctx->force_nb64 = (op == 1 || op == 6);
    if (op == 1) potrf_lower(ctx, A.p, n, n, info.p);
    TLG_CUDA(cudaEventRecord(e0, s));
    if (op == 0 || op == 6) potrf_lower(ctx, A.p, n, n, info.p);
    else if (op == 5) potrf_lower(ctx, A.p, n, n, info.p, B.p, n);
    else if (op == 1) trsm_left_lower(ctx, A.p, n, n, B.p, nrhs, n, 0);
    else if (op == 2) gemm(ctx, GemmDesc{n, nrhs, n, A.p, n, 0, A.p, n, 1, B.p, n, 1.0, 0.0, 0});
    else if (op == 3) {
      const int sm = sizeof(double) * std::max(kDiagSmemDoubles, 2 * 64 * 65 + 64 + 256);
      TLG_CUDA(cudaFuncSetAttribute(k_diag_tile_only, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      k_diag_tile_only<<<1, 128, sm, s>>>(A.p, n, B.p, info.p, nrhs);
    }
    else {
      int reps = nrhs;
      void* args[] = {&reps};
      TLG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_gridsync_only), dim3(n),
                                           dim3(128), args, 0, s));
    }
    TLG_CUDA(cudaEventRecord(e1, s));
    TLG_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    TLG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    best = std::min(best, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ctx->force_nb64 = false;
  return best;
}

bool debug_potrf(tlg_ctx* ctx, int n, const double* A, int tile, double* L, double* X, int band) {
  cudaStream_t s = ctx->stream;
  const size_t nn = static_cast<size_t>(n) * n;
  DBuf<double> dA, dX;
  dA.ensure(nn);
  dX.ensure(nn);
  DBuf<int> info;
  info.ensure(1);
  TLG_CUDA(cudaMemsetAsync(info.p, 0, sizeof(int), s));
  TLG_CUDA(cudaMemcpyAsync(dA.p, A, nn * 8, cudaMemcpyHostToDevice, s));
  ctx->force_nb64 = (tile == 64);
  if (tile == 32) {
    potrf_lower32(ctx, dA.p, n, n, info.p, dX.p, n, band);
  } else {
    potrf_lower(ctx, dA.p, n, n, info.p, dX.p, n, band);
  }
  ctx->force_nb64 = false;
  k_zero_upper<<<256, 256, 0, s>>>(dA.p, n);
  TLG_LAUNCHED(ctx);
  int h = 0;
  TLG_CUDA(cudaMemcpyAsync(&h, info.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  if (L) TLG_CUDA(cudaMemcpyAsync(L, dA.p, nn * 8, cudaMemcpyDeviceToHost, s));
  if (X) TLG_CUDA(cudaMemcpyAsync(X, dX.p, nn * 8, cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
  return h == 0;
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
  const unsigned b = static_cast<unsigned>(std::min<long long>((tot + 255) / 256, 4 * 148));
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
