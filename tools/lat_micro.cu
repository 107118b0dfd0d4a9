// Latency microbenchmark: dependent DFMA chain, double rsqrt, sqrt, div,
// __syncthreads with 4 warps, shared-memory round trip (cycles per op).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double seed) {
  __shared__ double sh[256];
  double a = seed + threadIdx.x, b = 1.0000001, c = 1e-9;
  long long t0, t1;
  const int N = 1024;
  t0 = clock64();
  for (int i = 0; i < N; ++i) a = fma(a, b, c);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) a = rsqrt(a) + 1.0;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) a = sqrt(a) + 1.0;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) a = 1.0 / a + 1.0;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0) / N;
  sh[threadIdx.x] = a;
  __syncthreads();
  t0 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < N; ++i) { double v = sh[idx]; idx = (int)v & 127; sh[idx] = v + 1.0; }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0) / N;
  // throughput: 8 independent chains
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = a + j;
  t0 = clock64();
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = fma(r[j], b, c);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = (t1 - t0) * 100 / (N * 8);
  double s = 0; for (int j = 0; j < 8; ++j) s += r[j];
  out[threadIdx.x] = a + s;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64 * 8);
  for (int nt : {32, 128}) {
    k<<<1, nt>>>(o, c, 1.0); cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, c, 7 * 8, cudaMemcpyDeviceToHost);
    printf("threads=%d dfma_lat=%lld rsqrt=%lld sqrt=%lld div=%lld syncthreads=%lld lds_sts_rt=%lld dfma_issue_x100=%lld\n",
           nt, h[0], h[1], h[2], h[3], h[4], h[5], h[6]);
  }
  return 0;
}
