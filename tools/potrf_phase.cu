// Per-phase wall time of the cooperative tile Cholesky (block 0's view):
// diag tile, panel (+X finalise), trailing (+X update) per 64-step.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//   -I paper_2509_26222_b200/csrc -I include tools/potrf_phase.cu -o build/potrf_phase
__device__ unsigned long long g_marks[3 * 1024];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TLG_COOP_MARK(k, step)                                        \
  do {                                                                \
    if (blockIdx.x == 0 && threadIdx.x == 0) g_marks[(step) * 3 + (k)] = gtime(); \
  } while (0)
#include "../paper_2509_26222_b200/csrc/dense.cu"
#include <cstdio>
#include <cstdlib>
#include <vector>
namespace tlg {
// SPD test matrix: n on the diagonal plus symmetric noise in [-0.5, 0.5)
__global__ void k_spd_fill(double* A, int n, unsigned seed) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * n;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(e % n), c = static_cast<int>(e / n);
    const int lo = min(r, c), hi = max(r, c);
    const unsigned hsh = (lo * 2654435761u) ^ (hi * 40503u) ^ seed;
    A[e] = (r == c ? n : 0.0) + ((hsh % 1000) / 1000.0 - 0.5);
  }
}
void throw_cuda(cudaError_t e, const char* w, const char* f, int l) {
  printf("cuda error %s at %s:%d (%s)\n", cudaGetErrorString(e), f, l, w);
  abort();
}
}
int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 400;
  const int withx = argc > 2 ? atoi(argv[2]) : 1;
  const int band = argc > 3 ? atoi(argv[3]) : -1;
  tlg_ctx ctx;
  cudaStreamCreate(&ctx.stream);
  cudaDeviceGetAttribute(&ctx.num_sms, cudaDevAttrMultiProcessorCount, 0);
  double *A, *X;
  int* info;
  cudaMalloc(&A, sizeof(double) * n * n);
  cudaMalloc(&X, sizeof(double) * n * n);
  cudaMalloc(&info, 4);
  for (int it = 0; it < 3; ++it) {
    tlg::k_spd_fill<<<256, 256, 0, ctx.stream>>>(A, n, 7u);
    tlg::potrf_lower(&ctx, A, n, n, info, withx ? X : nullptr, n, band);
    cudaStreamSynchronize(ctx.stream);
  }
  const int nt = (n <= 1024 || band > 0) ? (n + 31) / 32 : (n + 63) / 64;
  std::vector<unsigned long long> m(3 * nt);
  cudaMemcpyFromSymbol(m.data(), g_marks, sizeof(unsigned long long) * 3 * nt);
  double tot = 0, sd = 0, sp = 0, st = 0;
  for (int k = 0; k < nt; ++k) {
    const double d = (m[3 * k + 1] - m[3 * k]) * 1e-3, p = (m[3 * k + 2] - m[3 * k + 1]) * 1e-3;
    const double t = k + 1 < nt ? (m[3 * k + 3] - m[3 * k + 2]) * 1e-3 : 0;
    tot += d + p + t; sd += d; sp += p; st += t;
    if (k < 4 || k + 3 > nt || k % 16 == 0) printf("step %3d: diag %6.2f  panel %6.2f  trailing %6.2f us\n", k, d, p, t);
  }
  printf("sums: diag %.1f panel %.1f trailing %.1f us\n", sd, sp, st);
  printf("n=%d X=%d band=%d total(marks) %.1f us err=%s\n", n, withx, band, tot, cudaGetErrorString(cudaGetLastError()));
}
