// Do DFMA (FP64 pipe) and DMMA (tensor pipe, m8n8k4 f64) run concurrently on
// sm_100a? Times each alone and a mix where even warps run DFMA chains and odd
// warps run DMMA chains. nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dfma_loop(double* out, int iters) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-9 + k * 1e-9;
  const double b = 0.999999999, c = 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;
}
__device__ __forceinline__ void dmma_loop(double* out, int iters) {
  double c[8][2];
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0;
  const double a = 1e-3 * (threadIdx.x & 7), b = 2e-3 * (threadIdx.x & 3);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}
__global__ void k_mix(double* out, int mode, int it_f, int it_m) {
  const int w = threadIdx.x >> 5;
  if (mode == 0) dfma_loop(out, it_f);
  else if (mode == 1) dmma_loop(out, it_m);
  else if (w & 1) dmma_loop(out, it_m);
  else dfma_loop(out, it_f);
}
int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, it_f = 2048, it_m = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode) {
    k_mix<<<blocks, threads>>>(out, mode, 16, 32);
    cudaEventRecord(e0);
    k_mix<<<blocks, threads>>>(out, mode, it_f, it_m);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = blocks * threads / 32.0;
    const double f_flop = 2.0 * 32 * it_f * 16 * 8 * (mode == 0 ? warps : (mode == 2 ? warps / 2 : 0));
    const double m_flop = 512.0 * it_m * 8 * (mode == 1 ? warps : (mode == 2 ? warps / 2 : 0));
    printf("mode %d (%s): %.3f ms  DFMA %.1f TF/s  DMMA %.1f TF/s  total %.1f TF/s\n", mode,
           mode == 0 ? "DFMA only" : mode == 1 ? "DMMA only" : "half/half", ms,
           f_flop / (ms * 1e-3) / 1e12, m_flop / (ms * 1e-3) / 1e12,
           (f_flop + m_flop) / (ms * 1e-3) / 1e12);
  }
  return 0;
}
