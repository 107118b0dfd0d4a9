// Dense FP64 building blocks for the kernel-matrix update (column-major).
#pragma once

#include "internal.cuh"

namespace tlg {

// C = alpha * op(A) op(B) + beta * C   (op = transpose when t* != 0)
// uplo = 1 skips CTA tiles strictly above the diagonal (SYRK-style updates);
// uplo = 2 declares A lower triangular (ta = 0): row tile m0 reads K < m0 + 64.
struct GemmDesc {
  int M, N, K;
  const double* A;
  int lda, ta;
  const double* B;
  int ldb, tb;
  double* C;
  int ldc;
  double alpha, beta;
  int uplo;
};

void gemm(tlg_ctx* ctx, const GemmDesc& d);
// Grouped GEMM over `count` descriptors already resident in device memory.
// max_k > 512 lets long-K groups run split-K (uplo 0 descriptors only).
void gemm_grouped(tlg_ctx* ctx, const GemmDesc* d_descs, int count, int max_m, int max_n,
                  int max_k = 0);

// In-place lower Cholesky (A = L L^T) of the n x n matrix at A (lda).
// `info` (device int) is set non-zero when a pivot is not positive/finite.
// With X != nullptr the full inverse factor X = L^-1 (n x n, ldx, zero above
// the diagonal) is built in the same launch, so later solves are GEMMs.
// band < n declares A lower-banded (A_ij = 0 for i - j > band): the
// factorisation then skips the tiles outside the band (32-wide tiles).
void potrf_lower(tlg_ctx* ctx, double* A, int n, int lda, int* info, double* X = nullptr,
                 int ldx = 0, int band = -1);
// B <- L^-1 B (trans = 0) or B <- L^-T B (trans = 1); L lower n x n, B n x nrhs.
void trsm_left_lower(tlg_ctx* ctx, const double* L, int n, int ldl, double* B, int nrhs,
                     int ldb, int trans);
// potrf_lower with 32-wide tiles regardless of n (the banded path).
void potrf_lower32(tlg_ctx* ctx, double* A, int n, int lda, int* info, double* X, int ldx,
                   int band);
// x = (L L^T)^-1 b in place, L the (banded) 32-wide factor from the last
// potrf_lower (band as passed to it).
void band_solve(tlg_ctx* ctx, const double* L, int n, int ld, int band, double* b);
// A <- 0.5 (A + A^T) for a square n x n matrix (in place).
void symmetrize(tlg_ctx* ctx, double* A, int n, int lda);
// A[i,i] += v
void add_diag(tlg_ctx* ctx, double* A, int n, int lda, double v);

}  // namespace tlg
