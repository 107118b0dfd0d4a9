// Phase timing of warp_potrf_inv32 (one warp): load, factor, L store, X, linv store.
__device__ long long g_ph[16];
__shared__ long long s_ph[16];
__shared__ long long s_last;
#define TLG_PHASE(k)                                           \
  do {                                                         \
    if (threadIdx.x == 0) {                                    \
      long long _c = clock64();                                \
      s_ph[k] += _c - s_last;                                  \
      s_last = _c;                                             \
    }                                                          \
  } while (0)
#include "../paper_2509_26222_b200/csrc/dense.cu"
#include <cstdio>
#include <cstdlib>
namespace tlg {
void throw_cuda(cudaError_t e, const char*, const char*, int) { printf("cuda error %d\n", (int)e); abort(); }
}
__global__ void kk(double* A, double* linv, int* info, int reps) {
  __shared__ double sh[tlg::kWarpPotrfSmem];
  if (threadIdx.x == 0) for (int i = 0; i < 16; ++i) s_ph[i] = 0;
  __syncwarp();
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x == 0) s_last = clock64();
    __syncwarp();
    tlg::warp_potrf_inv32(A, 32, 32, linv, info, sh);
  }
  if (threadIdx.x == 0) for (int i = 0; i < 16; ++i) g_ph[i] = s_ph[i] / reps;
}
int main() {
  double h[32 * 32];
  for (int c = 0; c < 32; ++c) for (int r = 0; r < 32; ++r) h[r + 32 * c] = (r == c ? 32.0 : 0.0) + 0.01 * ((r * 7 + c * 3) % 11);
  for (int c = 0; c < 32; ++c) for (int r = 0; r < c; ++r) h[r + 32 * c] = h[c + 32 * r];
  double *A, *L; int* info;
  cudaMalloc(&A, sizeof h); cudaMalloc(&L, sizeof h); cudaMalloc(&info, 4);
  cudaMemcpy(A, h, sizeof h, cudaMemcpyHostToDevice);
  kk<<<1, 32>>>(A, L, info, 20);
  cudaDeviceSynchronize();
  long long p[16]; cudaMemcpyFromSymbol(p, g_ph, sizeof p);
  printf("cycles: load %lld factor %lld Lstore %lld X %lld linv %lld (err %s)\n", p[1], p[2], p[3], p[4], p[5],
         cudaGetErrorString(cudaGetLastError()));
}
