// Phase timing of tile_potrf_inv_la (clock64 at TLG_PHASE hooks: warp 0 vs worker warps)
// and the colown/rowown threads). nvcc ... -I paper_2509_26222_b200/csrc tools/diag_phase.cu
__device__ long long g_ph[16];
__shared__ long long s_ph[16];
__shared__ long long s_last[2];
#define TLG_PHASE(k)                                                     \
  do {                                                                   \
    if (threadIdx.x == 0 || threadIdx.x == 32) {                         \
      const int _w = threadIdx.x >> 5;                                   \
      long long _c = clock64();                                          \
      if (s_last[_w] != 0) s_ph[(k) + 8 * _w] += _c - s_last[_w];        \
      s_last[_w] = _c;                                                   \
    }                                                                    \
  } while (0)
#include "../paper_2509_26222_b200/csrc/dense.cu"
#include <cstdio>
#include <cstdlib>
namespace tlg {
void throw_cuda(cudaError_t e, const char*, const char*, int) { printf("cuda error %d\n", (int)e); abort(); }
}
__global__ void kk(double* A, double* linv, int* info, long long* tot) {
  extern __shared__ double shd[];
  if (threadIdx.x == 0) { s_last[0] = s_last[1] = 0; for (int i = 0; i < 16; ++i) s_ph[i] = 0; }
  __syncthreads();
  long long t0 = clock64();
  tlg::tile_potrf_inv_la(A, 64, 64, linv, info, shd);
  if (threadIdx.x == 0) { *tot = clock64() - t0; for (int i = 0; i < 16; ++i) g_ph[i] = s_ph[i]; }
}
int main() {
  double h[64 * 64];
  for (int c = 0; c < 64; ++c) for (int r = 0; r < 64; ++r) h[r + 64 * c] = (r == c ? 64.0 : 0.0) + 0.01 * ((r * 7 + c * 3) % 11);
  for (int c = 0; c < 64; ++c) for (int r = 0; r < c; ++r) h[r + 64 * c] = h[c + 64 * r];
  double *A, *L; int* info; long long* tot;
  cudaMalloc(&A, sizeof h); cudaMalloc(&L, sizeof h); cudaMalloc(&info, 4); cudaMalloc(&tot, 8);
  const int sm = sizeof(double) * tlg::kDiagSmemDoubles;
  cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  for (int it = 0; it < 3; ++it) {
    long long z[8] = {0}; cudaMemcpyToSymbol(g_ph, z, sizeof z);
    cudaMemcpy(A, h, sizeof h, cudaMemcpyHostToDevice);
    kk<<<1, 128, sm>>>(A, L, info, tot); cudaDeviceSynchronize();
    long long p[16], t; cudaMemcpyFromSymbol(p, g_ph, sizeof p); cudaMemcpy(&t, tot, 8, cudaMemcpyDeviceToHost);
    printf("warp0: update=%lld D=%lld factor=%lld Lrows=%lld Xrows=%lld wait=%lld | warp1: work=%lld wait=%lld\n", p[1], p[2], p[3], p[4], p[6], p[0], p[14], p[8]);
    printf("total=%lld cyc  update+stage=%lld sync1=%lld  4x4+panel=%lld  sync2=%lld  tail=%lld (err %s)\n", t, p[0], p[1], p[2], p[3], p[4],
           cudaGetErrorString(cudaGetLastError()));
  }
}
