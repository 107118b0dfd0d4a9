// FP64 roofline microbenchmark (tlg_measure_fp64_peak): sustained DFMA and
// DMMA throughput on the context's device, used as the FP64 denominator of
// the update's roofline (MEASURED_PEAKS.json has no FP64 entry).
#include "internal.cuh"

namespace tlg {

void prof_begin(tlg_ctx* ctx, int kernel) {
  if (!ctx->profiling) return;
  if (!ctx->prof_ev[0]) {
    TLG_CUDA(cudaEventCreate(&ctx->prof_ev[0]));
    TLG_CUDA(cudaEventCreate(&ctx->prof_ev[1]));
  }
  TLG_CUDA(cudaEventRecord(ctx->prof_ev[0], ctx->stream));
  ctx->prof_pending = kernel;
}

void prof_mark_end(tlg_ctx* ctx) {
  if (!ctx->profiling || ctx->prof_pending < 0) return;
  TLG_CUDA(cudaEventRecord(ctx->prof_ev[1], ctx->stream));
}

void prof_collect(tlg_ctx* ctx) {
  if (!ctx->profiling || ctx->prof_pending < 0) return;
  TLG_CUDA(cudaEventSynchronize(ctx->prof_ev[1]));
  float ms = 0.f;
  TLG_CUDA(cudaEventElapsedTime(&ms, ctx->prof_ev[0], ctx->prof_ev[1]));
  ctx->prof_ms[ctx->prof_pending] += ms;
  ctx->prof_n[ctx->prof_pending] += 1;
  ctx->prof_pending = -1;
}

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

}  // namespace tlg
