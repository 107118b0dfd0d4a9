// Batch-predict consumers either side of the update:
//   select_ground_points  (pipeline.cpp:150-170): ground-labelled scan points
//     moved to the world frame, ROI / radius filtered, first point per xy
//     voxel in scan order, capped at max_points;
//   terrain_error_histogram (metrics.cpp:199-232): |z - f(xy)| (0.25 m when
//     unsupported), sorted, top trim_fraction dropped, binned over [0, 0.25].
// Integer results (kept points, their order, bin counts) are bit-exact: the
// transform, norm and voxel keys use the reference's unfused expression order,
// first-in-voxel is a stable radix sort on the keys, bins are integer
// atomics on floor(e / 0.25 * bins) of the same doubles.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <cmath>
#include <vector>

#include "internal.cuh"

namespace tlg {

void eval_device(tlg_model* m, const double* x, const double* y, size_t n, double* z,
                 uint8_t* sup, double* gx, double* gy);

namespace {

struct Pose3 {
  double R[9];  // row-major
  double t[3];
};

constexpr uint64_t kNoKey = ~0ull;

// p = R f + t with Eigen's coefficient order (row dot product left to right,
// no FMA), then the ROI test (types.hpp:18-21), the radius test on the
// Euclidean norm and the voxel key (pipeline.cpp:157-164).
__global__ void k_ground_keys(const double* __restrict__ px, const double* __restrict__ py,
                              const double* __restrict__ pz, const uint8_t* __restrict__ kind,
                              size_t n, Pose3 pose, double rx0, double ry0, double rx1,
                              double ry1, double radius, double voxel,
                              uint64_t* __restrict__ keys, uint32_t* __restrict__ idx,
                              double* __restrict__ qx, double* __restrict__ qy,
                              double* __restrict__ qz) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  idx[i] = static_cast<uint32_t>(i);
  const double* R = pose.R;
  const double f0 = px[i], f1 = py[i], f2 = pz[i];
  const double x = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(R[0], f0), __dmul_rn(R[1], f1)),
                                       __dmul_rn(R[2], f2)), pose.t[0]);
  const double y = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(R[3], f0), __dmul_rn(R[4], f1)),
                                       __dmul_rn(R[5], f2)), pose.t[1]);
  const double z = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(R[6], f0), __dmul_rn(R[7], f1)),
                                       __dmul_rn(R[8], f2)), pose.t[2]);
  qx[i] = x;
  qy[i] = y;
  qz[i] = z;
  bool ok = kind[i] == 2;  // FeatureKind::Ground
  ok = ok && x >= rx0 && x <= rx1 && y >= ry0 && y <= ry1;
  const double dx = __dsub_rn(x, pose.t[0]), dy = __dsub_rn(y, pose.t[1]);
  ok = ok && !(__dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy))) > radius);
  uint64_t key = kNoKey;
  if (ok) {
    const int64_t vx = static_cast<int64_t>(floor(__ddiv_rn(x, voxel)));
    const int64_t vy = static_cast<int64_t>(floor(__ddiv_rn(y, voxel)));
    const int64_t k = static_cast<int64_t>(static_cast<uint64_t>(vx) << 21) ^
                      (vy & ((int64_t{1} << 21) - 1));
    key = static_cast<uint64_t>(k) ^ (1ull << 63);  // signed order as unsigned
  }
  keys[i] = key;
}

// sorted run heads = first point (lowest scan index, the sort is stable) of
// each voxel
__global__ void k_first_in_voxel(const uint64_t* __restrict__ keys,
                                 const uint32_t* __restrict__ idx, size_t n,
                                 uint8_t* __restrict__ keep) {
  const size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint64_t k = keys[p];
  if (k != kNoKey && (p == 0 || keys[p - 1] != k)) keep[idx[p]] = 1;
}

__global__ void k_gather3(const uint32_t* __restrict__ sel, size_t cnt,
                          const double* __restrict__ qx, const double* __restrict__ qy,
                          const double* __restrict__ qz, double* __restrict__ ox,
                          double* __restrict__ oy, double* __restrict__ oz) {
  const size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (j >= cnt) return;
  const uint32_t i = sel[j];
  if (ox) ox[j] = qx[i];
  if (oy) oy[j] = qy[i];
  if (oz) oz[j] = qz[i];
}

// |z - f| or kRange when unsupported (metrics.cpp:215-218), as sortable bits
__global__ void k_abs_errors(const double* __restrict__ z, const double* __restrict__ zp,
                             const uint8_t* __restrict__ sup, size_t n,
                             uint64_t* __restrict__ bits) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double e = sup[i] ? fabs(__dsub_rn(z[i], zp[i])) : 0.25;
  bits[i] = __double_as_longlong(e);  // e >= 0 (+0.0 from fabs): bit order = value order
}

__global__ void k_error_bins(const uint64_t* __restrict__ bits, size_t keep, int bins,
                             unsigned long long* __restrict__ counts) {
  extern __shared__ unsigned long long hist[];  // bins + 1 (last = overflow)
  for (int b = threadIdx.x; b <= bins; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < keep;
       i += (size_t)gridDim.x * blockDim.x) {
    const double e = __longlong_as_double(static_cast<long long>(bits[i]));
    const double fb = floor(__dmul_rn(__ddiv_rn(e, 0.25), static_cast<double>(bins)));
    atomicAdd(&hist[fb >= bins ? bins : static_cast<int>(fb)], 1ull);
  }
  __syncthreads();
  for (int b = threadIdx.x; b <= bins; b += blockDim.x)
    if (hist[b]) atomicAdd(&counts[b], hist[b]);
}

}  // namespace

size_t select_ground_device(tlg_ctx* ctx, const double* px, const double* py, const double* pz,
                            const uint8_t* kind, size_t n, const double R[9], const double t[3],
                            const double roi[4], double radius, double voxel, size_t max_points,
                            double* ox, double* oy, double* oz) {
  cudaStream_t s = ctx->stream;
  if (n == 0 || max_points == 0) return 0;
  require(n < (size_t{1} << 32), TLG_INVALID_ARGUMENT, "scan too large (2^32 points)");
  Pose3 pose;
  for (int i = 0; i < 9; ++i) pose.R[i] = R[i];
  for (int i = 0; i < 3; ++i) pose.t[i] = t[i];
  uint64_t* keys = ctx->ws<uint64_t>(S_KEYS, n);
  uint64_t* keys2 = ctx->ws<uint64_t>(S_KEYS2, n);
  uint32_t* idx = ctx->ws<uint32_t>(S_VALS, n);
  uint32_t* idx2 = ctx->ws<uint32_t>(S_VALS2, n);
  double* q = ctx->ws<double>(S_WORK1, 3 * n);
  uint8_t* keep = ctx->ws<uint8_t>(S_NODE_FLAG, n);
  uint32_t* sel = ctx->ws<uint32_t>(S_NODE_IDX, n);
  const unsigned nb = static_cast<unsigned>((n + 255) / 256);
  k_ground_keys<<<nb, 256, 0, s>>>(px, py, pz, kind, n, pose, roi[0], roi[1], roi[2], roi[3],
                                   radius, voxel, keys, idx, q, q + n, q + 2 * n);
  TLG_LAUNCHED(ctx);
  size_t tmp = 0;
  TLG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, keys2, idx, idx2, n, 0, 64, s));
  void* dtmp = ctx->ws<char>(S_CUB, tmp);
  TLG_CUDA(cub::DeviceRadixSort::SortPairs(dtmp, tmp, keys, keys2, idx, idx2, n, 0, 64, s));
  TLG_CUDA(cudaMemsetAsync(keep, 0, n, s));
  k_first_in_voxel<<<nb, 256, 0, s>>>(keys2, idx2, n, keep);
  TLG_LAUNCHED(ctx);
  int* d_cnt = ctx->ws<int>(S_COUNT, 1);
  thrust::counting_iterator<uint32_t> it(0);
  size_t tmp2 = 0;
  TLG_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp2, it, keep, sel, d_cnt, n, s));
  void* dtmp2 = ctx->ws<char>(S_CUB2, tmp2);
  TLG_CUDA(cub::DeviceSelect::Flagged(dtmp2, tmp2, it, keep, sel, d_cnt, n, s));
  int cnt = 0;
  TLG_CUDA(cudaMemcpyAsync(&cnt, d_cnt, sizeof(int), cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
  const size_t out = std::min(static_cast<size_t>(cnt), max_points);
  if (out) {
    k_gather3<<<(unsigned)((out + 255) / 256), 256, 0, s>>>(sel, out, q, q + n, q + 2 * n, ox,
                                                             oy, oz);
    TLG_LAUNCHED(ctx);
  }
  return out;
}

void error_histogram_device(tlg_model* m, const double* x, const double* y, const double* z,
                            size_t n, double trim_fraction, int bins, double* edges,
                            uint64_t* counts, uint64_t* trimmed, uint64_t* overflow) {
  tlg_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  require(n > 0, TLG_INVALID_ARGUMENT, "histogram needs matched non-empty samples");
  require(trim_fraction >= 0.0 && trim_fraction < 1.0, TLG_INVALID_ARGUMENT,
          "trim_fraction must be in [0, 1)");
  require(bins > 0, TLG_INVALID_ARGUMENT, "bins must be positive");
  double* zp = ctx->ws<double>(S_OUT_Z, n);
  uint8_t* sup = ctx->ws<uint8_t>(S_OUT_SUP, n);
  eval_device(m, x, y, n, zp, sup, nullptr, nullptr);
  uint64_t* bits = ctx->ws<uint64_t>(S_KEYS, n);
  uint64_t* bits2 = ctx->ws<uint64_t>(S_KEYS2, n);
  const unsigned nb = static_cast<unsigned>((n + 255) / 256);
  k_abs_errors<<<nb, 256, 0, s>>>(z, zp, sup, n, bits);
  TLG_LAUNCHED(ctx);
  size_t tmp = 0;
  TLG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, bits, bits2, n, 0, 64, s));
  void* dtmp = ctx->ws<char>(S_CUB, tmp);
  TLG_CUDA(cub::DeviceRadixSort::SortKeys(dtmp, tmp, bits, bits2, n, 0, 64, s));
  // metrics.cpp:220-223
  const size_t keep =
      n - static_cast<size_t>(std::floor(trim_fraction * static_cast<double>(n)));
  unsigned long long* d_counts = ctx->ws<unsigned long long>(S_COUNT, bins + 1);
  TLG_CUDA(cudaMemsetAsync(d_counts, 0, (bins + 1) * sizeof(unsigned long long), s));
  if (keep) {
    const unsigned hb = static_cast<unsigned>(std::min<size_t>((keep + 255) / 256, 2ull * ctx->num_sms));
    k_error_bins<<<hb, 256, (bins + 1) * sizeof(unsigned long long), s>>>(bits2, keep, bins,
                                                                         d_counts);
    TLG_LAUNCHED(ctx);
  }
  std::vector<unsigned long long> h(bins + 1);
  TLG_CUDA(cudaMemcpyAsync(h.data(), d_counts, (bins + 1) * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
  constexpr double kRange = 0.25;
  for (int b = 0; b <= bins; ++b) edges[b] = kRange * b / bins;  // metrics.cpp:226
  for (int b = 0; b < bins; ++b) counts[b] = h[b];
  *trimmed = n - keep;
  *overflow = h[bins];
}

}  // namespace tlg
