// Dependent-chain latencies (cycles per link) on one warp: DFMA, DMUL,
// rsqrt_pivot (MUFU.RSQ64H + third-order step), SHFL of a double,
// STS + __syncwarp + LDS of a double. nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// --expt-relaxed-constexpr -I include -I paper_2509_26222_b200/csrc tools/fp64_lat.cu
#include "../paper_2509_26222_b200/csrc/dense_tile.cuh"
#include <cstdio>
#include <cstdlib>
namespace tlg {
void throw_cuda(cudaError_t e, const char*, const char*, int) { printf("cuda error %d\n", (int)e); abort(); }
}
__device__ long long g_c[8];
__device__ double g_sink;
__global__ void kk(double seed, int n) {
  __shared__ double sm[64];
  const int lane = threadIdx.x & 31;
  double x = seed + lane * 1e-3;
  long long t0, t1;
  t0 = clock64();
  for (int r = 0; r < n; ++r) x = fma(x, 0.999999, 1e-9);
  t1 = clock64();
  if (lane == 0) g_c[0] = (t1 - t0) / n;
  t0 = clock64();
  for (int r = 0; r < n; ++r) x = x * 1.0000001;
  t1 = clock64();
  if (lane == 0) g_c[1] = (t1 - t0) / n;
  t0 = clock64();
  for (int r = 0; r < n; ++r) x = tlg::rsqrt_pivot(x) * x + 0.5;
  t1 = clock64();
  if (lane == 0) g_c[2] = (t1 - t0) / n;
  t0 = clock64();
  for (int r = 0; r < n; ++r) x = __shfl_sync(0xffffffffu, x, (r + 1) & 31);
  t1 = clock64();
  if (lane == 0) g_c[3] = (t1 - t0) / n;
  t0 = clock64();
  for (int r = 0; r < n; ++r) {
    sm[lane] = x;
    __syncwarp();
    x = sm[(lane + 1) & 31];
    __syncwarp();
  }
  t1 = clock64();
  if (lane == 0) g_c[4] = (t1 - t0) / n;
  t0 = clock64();
  for (int r = 0; r < n; ++r) x = rsqrt(x) * x + 0.5;
  t1 = clock64();
  if (lane == 0) g_c[5] = (t1 - t0) / n;
  if (x == 12345.0) g_sink = x;
}
int main() {
  kk<<<1, 32>>>(2.0, 1000);
  cudaDeviceSynchronize();
  long long c[8]; cudaMemcpyFromSymbol(c, g_c, sizeof c);
  printf("DFMA %lld  DMUL %lld  rsqrt_pivot+fma %lld  SHFL %lld  STS/sync/LDS %lld  rsqrt()+fma %lld (%s)\n",
         c[0], c[1], c[2], c[3], c[4], c[5], cudaGetErrorString(cudaGetLastError()));
}
