// DIAGNOSTICS (libterralio_diag.so, include/terralio_diag.h) — not part of
// the product library or its C-ABI: the FP64 roofline microbenchmark (the
// DFMA / DMMA denominators of the update's roofline; MEASURED_PEAKS.json has
// no FP64 entry), a dense-solver microbenchmark and a factor-a-host-matrix
// hook for the dense-layer tests. Links against libterralio_gpu.so and uses
// its internal dense kernels.
#include <cooperative_groups.h>

#include "../../../include/terralio_diag.h"
#include "../dense.cuh"

namespace cg = cooperative_groups;

namespace tlg {

__global__ void k_dfma_peak(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9, a3 = a0 + 3e-9;
  double a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9, a7 = a0 + 7e-9;
  const double b = 0.999999999, c = 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma_peak(double* out, int iters) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  const double a = 1e-3 * (threadIdx.x & 7), b = 2e-3 * (threadIdx.x & 3);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

void fp64_peak(tlg_ctx* ctx, double* dfma, double* dmma) {
  double* scratch = ctx->ws<double>(S_PARTIALS, 4);
  cudaEvent_t e0, e1;
  TLG_CUDA(cudaEventCreate(&e0));
  TLG_CUDA(cudaEventCreate(&e1));
  const int blocks = ctx->num_sms * 8, threads = 256;
  const int it_f = 4096, it_m = 8192;
  float ms = 0.f;
  k_dfma_peak<<<blocks, threads, 0, ctx->stream>>>(scratch, 64);  // warm-up
  TLG_CUDA(cudaEventRecord(e0, ctx->stream));
  k_dfma_peak<<<blocks, threads, 0, ctx->stream>>>(scratch, it_f);
  TLG_CUDA(cudaEventRecord(e1, ctx->stream));
  TLG_CUDA(cudaEventSynchronize(e1));
  TLG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  *dfma = 2.0 * blocks * threads * (double)it_f * 16 * 8 / (ms * 1e-3) / 1e12;
  k_dmma_peak<<<blocks, threads, 0, ctx->stream>>>(scratch, 64);
  TLG_CUDA(cudaEventRecord(e0, ctx->stream));
  k_dmma_peak<<<blocks, threads, 0, ctx->stream>>>(scratch, it_m);
  TLG_CUDA(cudaEventRecord(e1, ctx->stream));
  TLG_CUDA(cudaEventSynchronize(e1));
  TLG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  // one m8n8k4 per warp = 8*8*4 FMAs = 512 flop
  *dmma = 512.0 * (blocks * threads / 32) * (double)it_m * 8 / (ms * 1e-3) / 1e12;
  ctx->launches += 4;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
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

// Dense-layer microbenchmark: op 0 = Cholesky, 1 = trsm with nrhs columns,
// 2 = GEMM n x nrhs x n, 4 = grid barrier, 5 = Cholesky + X = L^-1,
// 6 = 64-wide Cholesky; best of `reps`, ms.
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

}  // namespace tlg

using namespace tlg;

namespace {
template <class F>
tlg_status diag_guard(F&& f) {
  try {
    f();
    return TLG_OK;
  } catch (const Error& e) {
    return e.status;
  } catch (...) {
    return TLG_RUNTIME_ERROR;
  }
}
}  // namespace

extern "C" {

tlg_status tlg_diag_fp64_peak(tlg_ctx* ctx, double* dfma, double* dmma) {
  return diag_guard([&] {
    double a = 0, b = 0;
    fp64_peak(ctx, &a, &b);
    if (dfma) *dfma = a;
    if (dmma) *dmma = b;
  });
}

tlg_status tlg_diag_dense_bench(tlg_ctx* ctx, int op, int n, int nrhs, int reps, double* ms) {
  return diag_guard([&] { *ms = dense_bench(ctx, op, n, nrhs, reps); });
}

tlg_status tlg_diag_potrf(tlg_ctx* ctx, int n, const double* A, int tile, int band, double* L,
                          double* X) {
  return diag_guard([&] {
    require(n > 0, TLG_INVALID_ARGUMENT, "n must be positive");
    require(tile == 0 || tile == 32 || tile == 64, TLG_INVALID_ARGUMENT, "tile must be 0, 32 or 64");
    if (!debug_potrf(ctx, n, A, tile, L, X, band > 0 && band < n ? band : n))
      throw Error(TLG_DOMAIN_ERROR, "matrix is not positive definite");
  });
}

tlg_status tlg_diag_set_batch_gram(tlg_model* m, int csr) {
  return diag_guard([&] {
    require(m != nullptr, TLG_INVALID_ARGUMENT, "null model");
    m->batch_csr_gram = csr != 0;
  });
}

tlg_status tlg_diag_last_gram_lattice(const tlg_model* m, int* lattice) {
  return diag_guard([&] {
    require(m != nullptr && lattice != nullptr, TLG_INVALID_ARGUMENT, "null argument");
    *lattice = m->last_gram_lattice;
  });
}

}  // extern "C"
