// Per-kernel CUDA-event timing of the hot kernels (tlg_ctx_set_profiling /
// tlg_ctx_kernel_stats: bench.py reads the kernel's own average duration).
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

}  // namespace tlg
