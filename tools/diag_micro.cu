// Standalone microbenchmark of the 64x64 diagonal-tile factorisation phases.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/diag_micro.cu -o build/diag_micro
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(128) k(double* A, double* out, int reps, long long* cyc) {
  __shared__ double a[64][65];
  __shared__ double isd[64];
  const int t = threadIdx.x;
  long long t0 = clock64();
  double acc = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int e = t; e < 64 * 64; e += 128) {
      const int r = e & 63, c = e >> 6;
      a[r][c] = A[r + c * 64];
    }
    __syncthreads();
    if (MODE >= 1) {
      const int p = t & 31, cp = t >> 5;
#pragma unroll 1
      for (int j = 0; j < 64; ++j) {
        double d = a[j][j];
        if (MODE >= 2) {
          const double is = rsqrt(d);
          if (t == 0) isd[j] = is;
          d = is * is;
        }
        if (MODE >= 3) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = h ? 63 - p : p;
            if (r > j) {
              const double f = a[r][j] * d;
              for (int c = j + 1 + ((cp - j - 1) & 3); c <= r; c += 4)
                a[r][c] = fma(-f, a[c][j], a[r][c]);
            }
          }
        }
        acc += d;
        __syncthreads();
      }
    }
    for (int e = t; e < 64 * 64; e += 128) {
      const int r = e & 63, c = e >> 6;
      out[r + c * 64] = a[r][c] + acc;
    }
    __syncthreads();
  }
  if (t == 0) *cyc = clock64() - t0;
}

int main() {
  double *A, *out;
  long long* cyc;
  cudaMalloc(&A, 64 * 64 * 8);
  cudaMalloc(&out, 64 * 64 * 8);
  cudaMalloc(&cyc, 8);
  double h[64 * 64];
  for (int i = 0; i < 64; ++i)
    for (int j = 0; j < 64; ++j) h[i + j * 64] = (i == j ? 64.0 : 0.0) + 0.01 * ((i * 7 + j * 3) % 11);
  cudaMemcpy(A, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, const char* name) {
    kern<<<1, 128>>>(A, out, 2, cyc);
    cudaEventRecord(e0);
    kern<<<1, 128>>>(A, out, 20, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %8.2f us/rep  %10lld cycles/rep  err=%s\n", name, ms * 1e3 / 20, c / 20,
           cudaGetErrorString(cudaGetLastError()));
  };
  run(k<0>, "load+store only");
  run(k<1>, "+64 pivots (sync only)");
  run(k<2>, "+rsqrt per pivot");
  run(k<3>, "+trailing update");
  return 0;
}
