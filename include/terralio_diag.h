/* terralio_diag.h — DIAGNOSTICS, not the product ABI (libterralio_diag.so,
 * built from paper_2509_26222_b200/csrc/diag/diag.cu against
 * libterralio_gpu.so). Used by bench.py (the FP64 roofline denominators),
 * the dense-layer tests and tools/. */
#ifndef TERRALIO_DIAG_H_
#define TERRALIO_DIAG_H_

#include "terralio_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Sustained DFMA and DMMA (mma.sync m8n8k4 f64) TFLOP/s on ctx's device. */
tlg_status tlg_diag_fp64_peak(tlg_ctx* ctx, double* dfma_tflops, double* dmma_tflops);
/* Dense-solver microbenchmark: op 0 = Cholesky of an n x n SPD matrix,
 * 1 = triangular solve with nrhs right-hand sides, 2 = GEMM n x nrhs x n,
 * 4 = grid barrier (nrhs repetitions), 5 = Cholesky + inverse factor,
 * 6 = 64-wide Cholesky. Best of `reps`, ms. */
tlg_status tlg_diag_dense_bench(tlg_ctx* ctx, int op, int n, int nrhs, int reps, double* ms);
/* Factor the host SPD matrix A (n x n, column-major) with the device
 * Cholesky (tile 0 = automatic, 32, 64; band < n declares it banded) and
 * return L and X = L^-1 (host, may be NULL). */
tlg_status tlg_diag_potrf(tlg_ctx* ctx, int n, const double* A, int tile, int band, double* L,
                          double* X);
/* Batch-ridge assembly path of model m: 0 = automatic (the lattice element
 * assembly when the centres are mesh nodes), 1 = the row-wise CSR Gram
 * always (the A/B reference for the lattice path). */
tlg_status tlg_diag_set_batch_gram(tlg_model* m, int csr);
/* 1 when m's most recent Gram assembly (batch ridge, information-form
 * update) took the lattice element path, else 0. */
tlg_status tlg_diag_last_gram_lattice(const tlg_model* m, int* lattice);

#ifdef __cplusplus
}
#endif

#endif /* TERRALIO_DIAG_H_ */
