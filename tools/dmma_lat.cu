// DMMA (mma.sync m8n8k4 f64) latency / per-warp throughput with 1..16 independent chains.
#include <cstdio>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int C>
__global__ void k(double* out, long long* cyc) {
  double acc[C][2];
  for (int i = 0; i < C; ++i) acc[i][0] = acc[i][1] = threadIdx.x + i * 1.5;
  double a = 1.0000001, b = 0.999999;
  const int N = 256;
  long long t0 = clock64();
  for (int it = 0; it < N; ++it)
#pragma unroll
    for (int i = 0; i < C; ++i) dmma(acc[i][0], acc[i][1], a + i, b - i);
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < C; ++i) s += acc[i][0] + acc[i][1];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = (t1 - t0) / N;
}
template <int C>
void run(double* o, long long* c, int warps) {
  k<C><<<1, 32 * warps>>>(o, c);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("chains=%2d warps=%d: %lld cycles per iteration (%.1f cycles per dmma per warp)\n", C, warps, h, (double)h / C);
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8);
  for (int w : {1, 4, 8}) { run<1>(o, c, w); run<4>(o, c, w); run<8>(o, c, w); run<16>(o, c, w); }
}
