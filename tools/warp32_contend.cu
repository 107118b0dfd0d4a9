// warp_potrf_inv32 (one warp, the K7f diagonal step) timed alone and with
// co-resident warps of the same CTA saturating the FP64 datapath with DMMA
// (mode 1: all 7 other warps, mode 2: only the one sharing warp 0's SMSP,
// mode 3: 7 warps of DFMA). nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// --expt-relaxed-constexpr -I include -I paper_2509_26222_b200/csrc tools/warp32_contend.cu
#include "../paper_2509_26222_b200/csrc/dense.cu"
#include <cstdio>
#include <cstdlib>
namespace tlg {
void throw_cuda(cudaError_t e, const char*, const char*, int) { printf("cuda error %d\n", (int)e); abort(); }
}
__device__ long long g_cyc;
__device__ double g_sink;
__global__ void kk(double* A, double* linv, int* info, int reps, int mode) {
  __shared__ double sh[tlg::kWarpPotrfSmem];
  __shared__ volatile int done;
  const int w = threadIdx.x >> 5;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  if (w == 0) {
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) tlg::warp_potrf_inv32(A, 32, 32, linv, info, sh);
    long long t1 = clock64();
    if (threadIdx.x == 0) { g_cyc = (t1 - t0) / reps; done = 1; }
  } else {
    const bool active = mode == 1 || mode == 3 || (mode == 2 && (w & 3) == 0);
    if (!active) return;
    double c0 = threadIdx.x, c1 = 1.0, a = 1.0000001, b = 0.9999999;
    double d[8] = {1, 2, 3, 4, 5, 6, 7, 8};
    while (!done) {
      for (int i = 0; i < 64; ++i) {
        if (mode == 3) {
#pragma unroll
          for (int q = 0; q < 8; ++q) d[q] = fma(d[q], a, b);
        } else {
          tlg::dmma(c0, c1, a, b);
        }
      }
    }
    double s = c0 + c1;
    for (int q = 0; q < 8; ++q) s += d[q];
    if (s == 12345.0) g_sink = s;
  }
}
int main() {
  double h[32 * 32];
  for (int c = 0; c < 32; ++c) for (int r = 0; r < 32; ++r) h[r + 32 * c] = (r == c ? 32.0 : 0.0) + 0.01 * ((r * 7 + c * 3) % 11);
  for (int c = 0; c < 32; ++c) for (int r = 0; r < c; ++r) h[r + 32 * c] = h[c + 32 * r];
  double *A, *L; int* info;
  cudaMalloc(&A, sizeof h); cudaMalloc(&L, sizeof h); cudaMalloc(&info, 4);
  const char* names[] = {"alone", "7 warps DMMA", "1 same-SMSP warp DMMA", "7 warps DFMA"};
  for (int mode = 0; mode < 4; ++mode) {
    cudaMemcpy(A, h, sizeof h, cudaMemcpyHostToDevice);
    kk<<<1, 256>>>(A, L, info, 20, mode);
    cudaDeviceSynchronize();
    long long c; cudaMemcpyFromSymbol(&c, g_cyc, sizeof c);
    printf("%-26s %lld cycles per factor+inverse (%s)\n", names[mode], c, cudaGetErrorString(cudaGetLastError()));
  }
}
