// Cycles per 64x64xK gemm_tile call inside one CTA (L2-resident operands).
#include "../paper_2509_26222_b200/csrc/dense.cu"
#include <cstdio>
#include <cstdlib>
namespace tlg {
void throw_cuda(cudaError_t e, const char*, const char*, int) { printf("cuda error %d\n", (int)e); abort(); }
}
template <int T32>
__global__ void __launch_bounds__(128) kk(tlg::GemmDesc d, int reps, long long* cyc) {
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (T32) tlg::gemm32_tile(d, 0, 0);
    else tlg::gemm_tile(d, 0, 0);
    __syncthreads();
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = (clock64() - t0) / reps;
}
int main() {
  double *A, *B, *C;
  long long* cyc;
  cudaMalloc(&A, 8 * 4096 * 64);
  cudaMalloc(&B, 8 * 4096 * 64);
  cudaMalloc(&C, 8 * 64 * 64 * 148);
  cudaMalloc(&cyc, 8 * 148);
  cudaMemset(A, 0, 8 * 4096 * 64);
  cudaMemset(B, 0, 8 * 4096 * 64);
  for (int K : {32, 64, 256}) {
    for (int ta = 0; ta < 2; ++ta) {
      tlg::GemmDesc d{64, 64, K, A, ta ? K : 64, ta, B, 64, 1, C, 64, -1.0, 1.0, 0};
      if (!ta) d.lda = 64;
      if (!ta) d.lda = 64, d.A = A;
      d.ldb = 64;
      for (int t32 = 0; t32 < 2; ++t32) {
        if (t32) kk<1><<<1, 128>>>(d, 50, cyc);
        else kk<0><<<1, 128>>>(d, 50, cyc);
        cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        const int T = t32 ? 32 : 64;
        printf("tile %d K=%4d ta=%d tb=1: %lld cycles/tile (%.2f us at 1.9GHz) %.1f flop/clk  err=%s\n", T, K, ta, c,
               c / 1900.0, 2.0 * T * T * K / c, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
}
