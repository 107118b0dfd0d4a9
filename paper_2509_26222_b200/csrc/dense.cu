// Dense FP64 kernels for the kernel-matrix update: a DMMA (mma.sync
// m8n8k4 f64, the sm_100a FP64 tensor path — tcgen05 has no f64 kind) GEMM
// with 64x64 CTA tiles, a blocked right-looking Cholesky (64-wide panels:
// single-CTA diagonal factor in shared memory, row-parallel panel solve,
// DMMA trailing update) and blocked triangular solves.
#include "dense.cuh"

namespace tlg {

constexpr int TM = 64, TN = 64, TK = 16, SP = 68;  // smem pitch (doubles): conflict-free frags

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void gemm_tile(const GemmDesc& d, int tile_m, int tile_n) {
  const int m0 = tile_m * TM, n0 = tile_n * TN;
  if (m0 >= d.M || n0 >= d.N) return;
  if (d.uplo == 1 && m0 + TM <= n0) return;  // strictly above the diagonal
  __shared__ double As[TK][SP];
  __shared__ double Bs[TK][SP];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int wm = (w & 1) * 32, wn = (w >> 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int k0 = 0; k0 < d.K; k0 += TK) {
    // A tile: op(A)(m0 + i, k0 + k) -> As[k][i]
    if (!d.ta) {
      const int i = t & 63;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int k = (t >> 6) + 2 * s;
        const int gi = m0 + i, gk = k0 + k;
        As[k][i] = (gi < d.M && gk < d.K) ? d.A[gi + (size_t)gk * d.lda] : 0.0;
      }
    } else {
      const int k = t & 15;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int i = (t >> 4) + 8 * s;
        const int gi = m0 + i, gk = k0 + k;
        As[k][i] = (gi < d.M && gk < d.K) ? d.A[gk + (size_t)gi * d.lda] : 0.0;
      }
    }
    // B tile: op(B)(k0 + k, n0 + j) -> Bs[k][j]
    if (!d.tb) {
      const int k = t & 15;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int j = (t >> 4) + 8 * s;
        const int gj = n0 + j, gk = k0 + k;
        Bs[k][j] = (gj < d.N && gk < d.K) ? d.B[gk + (size_t)gj * d.ldb] : 0.0;
      }
    } else {
      const int j = t & 63;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int k = (t >> 6) + 2 * s;
        const int gj = n0 + j, gk = k0 + k;
        Bs[k][j] = (gj < d.N && gk < d.K) ? d.B[gj + (size_t)gk * d.ldb] : 0.0;
      }
    }
    __syncthreads();
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
// Cholesky of one <=64 x 64 diagonal tile in shared memory (lower part).
constexpr int NB = 64;

__global__ void __launch_bounds__(256) k_potrf_tile(double* __restrict__ A, int lda, int kb,
                                                    int* __restrict__ info) {
  __shared__ double a[NB][NB + 1];
  const int t = threadIdx.x;
  for (int e = t; e < kb * kb; e += blockDim.x) {
    const int r = e % kb, c = e / kb;
    a[r][c] = (r >= c) ? A[r + (size_t)c * lda] : 0.0;
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
  for (int e = t; e < kb * kb; e += blockDim.x) {
    const int r = e % kb, c = e / kb;
    if (r >= c) A[r + (size_t)c * lda] = a[r][c];
  }
}

// P <- P L^-T for `rows` rows of P (row-parallel; L = kb x kb lower tile).
__global__ void __launch_bounds__(128) k_trsm_rows_lt(const double* __restrict__ L, int ldl,
                                                      int kb, double* __restrict__ P, int ldp,
                                                      int rows) {
  __shared__ double l[NB][NB + 1];
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
    const int r = e % kb, c = e / kb;
    l[r][c] = (r >= c) ? L[r + (size_t)c * ldl] : 0.0;
  }
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  double x[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c)
    if (c < kb) x[c] = P[i + (size_t)c * ldp];
  // x L^T = p  ->  x_c = (p_c - sum_{k<c} x_k l_ck) / l_cc
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    if (c < kb) {
      double s = x[c];
#pragma unroll
      for (int k = 0; k < NB; ++k)
        if (k < c) s = fma(-x[k], l[c][k], s);
      x[c] = s / l[c][c];
    }
  }
#pragma unroll
  for (int c = 0; c < NB; ++c)
    if (c < kb) P[i + (size_t)c * ldp] = x[c];
}

// B_k <- L_kk^-1 B_k (trans=0) or L_kk^-T B_k (trans=1): column-parallel,
// 32 columns per CTA staged through shared memory.
__global__ void __launch_bounds__(128) k_trsm_tile_cols(const double* __restrict__ L, int ldl,
                                                        int kb, double* __restrict__ B, int ldb,
                                                        int ncols, int trans) {
  __shared__ double l[NB][NB + 1];
  __shared__ double bs[NB][17];
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
    const int r = e % kb, c = e / kb;
    l[r][c] = (r >= c) ? L[r + (size_t)c * ldl] : 0.0;
  }
  const int c0 = blockIdx.x * 16;
  for (int e = threadIdx.x; e < kb * 16; e += blockDim.x) {
    const int r = e % kb, c = e / kb;
    bs[r][c] = (c0 + c < ncols) ? B[r + (size_t)(c0 + c) * ldb] : 0.0;
  }
  __syncthreads();
  // 4 threads per column: each owns a row quarter? keep it simple: 1 thread / column
  if (threadIdx.x < 16) {
    const int c = threadIdx.x;
    if (!trans) {
      for (int r = 0; r < kb; ++r) {
        double s = bs[r][c];
        for (int k = 0; k < r; ++k) s = fma(-l[r][k], bs[k][c], s);
        bs[r][c] = s / l[r][r];
      }
    } else {
      for (int r = kb - 1; r >= 0; --r) {
        double s = bs[r][c];
        for (int k = r + 1; k < kb; ++k) s = fma(-l[k][r], bs[k][c], s);
        bs[r][c] = s / l[r][r];
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kb * 16; e += blockDim.x) {
    const int r = e % kb, c = e / kb;
    if (c0 + c < ncols) B[r + (size_t)(c0 + c) * ldb] = bs[r][c];
  }
}

void potrf_lower(tlg_ctx* ctx, double* A, int n, int lda, int* info) {
  for (int k0 = 0; k0 < n; k0 += NB) {
    const int kb = std::min(NB, n - k0);
    double* Akk = A + k0 + (size_t)k0 * lda;
    k_potrf_tile<<<1, 256, 0, ctx->stream>>>(Akk, lda, kb, info);
    TLG_LAUNCHED(ctx);
    const int rows = n - k0 - kb;
    if (rows <= 0) break;
    double* P = A + (k0 + kb) + (size_t)k0 * lda;
    k_trsm_rows_lt<<<(rows + 127) / 128, 128, 0, ctx->stream>>>(Akk, lda, kb, P, lda, rows);
    TLG_LAUNCHED(ctx);
    GemmDesc d{rows, rows, kb, P, lda, 0, P, lda, 1,
               A + (k0 + kb) + (size_t)(k0 + kb) * lda, lda, -1.0, 1.0, 1};
    gemm(ctx, d);
  }
}

void trsm_left_lower(tlg_ctx* ctx, const double* L, int n, int ldl, double* B, int nrhs,
                     int ldb, int trans) {
  if (n <= 0 || nrhs <= 0) return;
  const int nblk = (n + NB - 1) / NB;
  if (!trans) {
    for (int kbi = 0; kbi < nblk; ++kbi) {
      const int k0 = kbi * NB, kb = std::min(NB, n - k0);
      if (k0 > 0) {  // B_k -= L[k, 0:k0] B[0:k0]
        GemmDesc d{kb, nrhs, k0, L + k0, ldl, 0, B, ldb, 0, B + k0, ldb, -1.0, 1.0, 0};
        gemm(ctx, d);
      }
      k_trsm_tile_cols<<<(nrhs + 15) / 16, 128, 0, ctx->stream>>>(L + k0 + (size_t)k0 * ldl, ldl,
                                                                  kb, B + k0, ldb, nrhs, 0);
      TLG_LAUNCHED(ctx);
    }
  } else {
    for (int kbi = nblk - 1; kbi >= 0; --kbi) {
      const int k0 = kbi * NB, kb = std::min(NB, n - k0);
      const int rest = n - k0 - kb;
      if (rest > 0) {  // B_k -= L[k0+kb:, k]^T B[k0+kb:]
        GemmDesc d{kb, nrhs, rest, L + (k0 + kb) + (size_t)k0 * ldl, ldl, 1, B + k0 + kb, ldb, 0,
                   B + k0, ldb, -1.0, 1.0, 0};
        gemm(ctx, d);
      }
      k_trsm_tile_cols<<<(nrhs + 15) / 16, 128, 0, ctx->stream>>>(L + k0 + (size_t)k0 * ldl, ldl,
                                                                  kb, B + k0, ldb, nrhs, 1);
      TLG_LAUNCHED(ctx);
    }
  }
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
