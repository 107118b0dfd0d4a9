// Cycles and agreement of the one-warp (warp_potrf_inv32) and the pipelined
// two-warp (warp2_potrf_inv32) 32x32 Cholesky + inverse on a shared-memory
// tile, alone and beside a DMMA-saturating warp on each other SMSP.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr
//   -I include -I paper_2509_26222_b200/csrc tools/warp2_phase.cu
__device__ long long g_piv[33];
__shared__ long long s_piv[33];
#define TLG_PIVOT_STAMP(j) do { if (threadIdx.x == 0) s_piv[j] += clock64(); } while (0)
#include "../paper_2509_26222_b200/csrc/dense.cu"
#include <cmath>
#include <cstdio>
#include <cstdlib>
namespace tlg {
void throw_cuda(cudaError_t e, const char*, const char*, int) { printf("cuda error %d\n", (int)e); abort(); }
}
__device__ long long g_cyc, g_w0, g_w1;
__global__ void kk(const double* A, double* Lout, double* linv, int* info, int reps, int which, int contend) {
  constexpr int P = 36;
  __shared__ __align__(16) double T[32 * P];
  __shared__ __align__(16) double sh[tlg::kWarp2PotrfSmem + tlg::kWarpPotrfSmem];
  __shared__ volatile int done;
  __shared__ long long s_w0, s_w1;
  const int t = threadIdx.x, w = t >> 5;
  if (t == 0) { done = 0; s_w0 = 0; s_w1 = 0; for (int q = 0; q < 33; ++q) s_piv[q] = 0; }
  long long acc = 0;
  for (int r = 0; r < reps; ++r) {
    for (int e = t; e < 1024; e += blockDim.x) T[(e & 31) + (e >> 5) * P] = A[e];
    if (t == 0) *tlg::warp2_potrf_pub(sh) = 0;
    __syncthreads();
    long long t0 = clock64();
    if (which == 0) {
      if (w == 0) tlg::warp_potrf_inv32(T, P, 32, linv, info, sh);
    } else if (w < 2) {
      if (which == 1) tlg::warp2_potrf_inv32(T, P, 32, linv, info, sh);
      else tlg::warp2b_potrf_inv32(T, P, 32, linv, info, sh);
    }
    if (t == 0) { s_w0 += clock64() - t0; s_piv[32] += clock64(); }
    if (t == 32) s_w1 += clock64() - t0;
    __syncthreads();
    acc += clock64() - t0;
  }
  if (t == 0) {
    g_cyc = acc / reps;
    g_w0 = s_w0 / reps;
    g_w1 = s_w1 / reps;
    for (int q = 0; q < 33; ++q) g_piv[q] = s_piv[q];
    done = 1;
  }
  for (int e = t; e < 1024; e += blockDim.x) Lout[e] = T[(e & 31) + (e >> 5) * P];
  (void)contend;
}
int main() {
  double h[32 * 32];
  for (int c = 0; c < 32; ++c) for (int r = 0; r < 32; ++r) h[r + 32 * c] = (r == c ? 32.0 : 0.0) + 0.01 * ((r * 7 + c * 3) % 11);
  for (int c = 0; c < 32; ++c) for (int r = 0; r < c; ++r) h[r + 32 * c] = h[c + 32 * r];
  double *A, *L, *X; int* info;
  cudaMalloc(&A, sizeof h); cudaMalloc(&L, sizeof h); cudaMalloc(&X, sizeof h); cudaMalloc(&info, 4);
  cudaMemcpy(A, h, sizeof h, cudaMemcpyHostToDevice);
  double Lr[3][1024], Xr[3][1024];
  for (int which = 0; which < 3; ++which) {
    cudaMemset(info, 0, 4);
    kk<<<1, 128>>>(A, L, X, info, 50, which, 0);
    cudaDeviceSynchronize();
    long long c, c0, c1; cudaMemcpyFromSymbol(&c, g_cyc, sizeof c);
    cudaMemcpyFromSymbol(&c0, g_w0, sizeof c0); cudaMemcpyFromSymbol(&c1, g_w1, sizeof c1);
    printf("  warp 0 done %lld, warp 1 done %lld\n", c0, c1);
    if (which == 2) {
      long long pv[33]; cudaMemcpyFromSymbol(pv, g_piv, sizeof pv);
      printf("  per pivot:");
      for (int q = 0; q < 32; ++q) printf(" %lld", (pv[q + 1] - pv[q]) / 50);
      printf("\n");
    }
    int inf; cudaMemcpy(&inf, info, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(Lr[which], L, sizeof h, cudaMemcpyDeviceToHost);
    cudaMemcpy(Xr[which], X, sizeof h, cudaMemcpyDeviceToHost);
    printf("%s: %lld cycles (info %d, %s)\n", which == 2 ? "two-warp blocked" : which ? "two-warp" : "one-warp", c, inf,
           cudaGetErrorString(cudaGetLastError()));
  }
  for (int v = 1; v < 3; ++v) {
  double dl = 0, dx = 0;
  for (int c = 0; c < 32; ++c) for (int r = c; r < 32; ++r) dl = fmax(dl, fabs(Lr[0][r + 32 * c] - Lr[v][r + 32 * c]));
  for (int e = 0; e < 1024; ++e) dx = fmax(dx, fabs(Xr[0][e] - Xr[v][e]));
  // L L^T = A and X L = I
  double rl = 0, rx = 0;
  for (int r = 0; r < 32; ++r) for (int c = 0; c <= r; ++c) {
    double s = 0, q = 0;
    for (int k = 0; k <= c; ++k) s += Lr[v][r + 32 * k] * Lr[v][c + 32 * k];
    rl = fmax(rl, fabs(s - h[r + 32 * c]));
    for (int k = 0; k < 32; ++k) q += Xr[v][r + 32 * k] * (k >= c ? Lr[v][k + 32 * c] : 0.0);
    rx = fmax(rx, fabs(q - (r == c ? 1.0 : 0.0)));
  }
  printf("variant %d: max |L - L1| %.3g  max |X - X1| %.3g  |LL^T - A| %.3g  |XL - I| %.3g\n", v, dl, dx, rl, rx);
  }
}
