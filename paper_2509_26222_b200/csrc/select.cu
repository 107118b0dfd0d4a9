// K2 select_centres: supported_mesh_nodes (center_select.cpp:18-62).
//
// Points are binned by the reference's GridIndex2 cell key
// (floor(v / max(r_a, res)), packed like grid_index.hpp:58-61) with a device
// radix sort; every lattice node of the ROI gets one thread that checks the
// dilated-bbox window (center_select.cpp:36-50), rebuilds the node
// coordinate exactly (min + i*res, no FMA) and counts points with
// r^2 <= r_a^2 in the (2 span + 1)^2 cells by binary search on the sorted
// keys. Nodes are compacted in (i outer, j inner) order -> bit-exact node
// list and order.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <cfloat>
#include <cmath>

#include "internal.cuh"

namespace tlg {

__device__ __forceinline__ uint64_t cell_key(int ix, int iy) {
  return (static_cast<uint64_t>(static_cast<uint32_t>(ix)) << 32) | static_cast<uint32_t>(iy);
}

__global__ void k_validate(const double* __restrict__ x, const double* __restrict__ y,
                           const double* __restrict__ z, size_t m, size_t zn,
                           int* __restrict__ err) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m;
       i += (size_t)gridDim.x * blockDim.x) {
    bool ok = isfinite(x[i]) && isfinite(y[i]);
    if (i < zn) ok = ok && isfinite(z[i]);
    if (!ok) atomicOr(err, 1);
  }
}

int* validate_obs_launch(tlg_ctx* ctx, const double* x, const double* y, const double* z,
                         size_t m, size_t zn) {
  // TerrainObservation::validate (center_select.cpp:9-16)
  if (m != zn) throw Error(TLG_INVALID_ARGUMENT, "observation xy/z length mismatch");
  if (m == 0) throw Error(TLG_INVALID_ARGUMENT, "empty observation");
  int* err = ctx->ws<int>(S_VALIDATE, 1);
  TLG_CUDA(cudaMemsetAsync(err, 0, sizeof(int), ctx->stream));
  const unsigned blocks = static_cast<unsigned>(std::min<size_t>((m + 255) / 256, 8ull * ctx->num_sms));
  k_validate<<<blocks, 256, 0, ctx->stream>>>(x, y, z, m, zn, err);
  TLG_LAUNCHED(ctx);
  return err;
}

void validate_obs_check(int flag) {
  if (flag) throw Error(TLG_INVALID_ARGUMENT, "non-finite observation coordinate");
}

void validate_obs_device(tlg_ctx* ctx, const double* x, const double* y, const double* z,
                         size_t m, size_t zn) {
  const int* err = validate_obs_launch(ctx, x, y, z, m, zn);
  int h = 0;
  TLG_CUDA(cudaMemcpyAsync(&h, err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  TLG_CUDA(cudaStreamSynchronize(ctx->stream));
  validate_obs_check(h);
}

// cell keys of the points + per-block bbox partials
__global__ void k_point_keys(const double* __restrict__ x, const double* __restrict__ y, size_t m,
                             double cell, uint64_t* __restrict__ key, uint32_t* __restrict__ idx,
                             double* __restrict__ bbox_part) {
  double mnx = DBL_MAX, mny = DBL_MAX, mxx = -DBL_MAX, mxy = -DBL_MAX;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m;
       i += (size_t)gridDim.x * blockDim.x) {
    const double px = x[i], py = y[i];
    key[i] = cell_key(static_cast<int>(floor(px / cell)), static_cast<int>(floor(py / cell)));
    idx[i] = static_cast<uint32_t>(i);
    mnx = fmin(mnx, px);
    mny = fmin(mny, py);
    mxx = fmax(mxx, px);
    mxy = fmax(mxy, py);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mnx = fmin(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
    mny = fmin(mny, __shfl_xor_sync(0xffffffffu, mny, o));
    mxx = fmax(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
    mxy = fmax(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
  }
  __shared__ double sh[4][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    sh[0][wid] = mnx;
    sh[1][wid] = mny;
    sh[2][wid] = mxx;
    sh[3][wid] = mxy;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      mnx = fmin(mnx, sh[0][w]);
      mny = fmin(mny, sh[1][w]);
      mxx = fmax(mxx, sh[2][w]);
      mxy = fmax(mxy, sh[3][w]);
    }
    bbox_part[blockIdx.x * 4 + 0] = mnx;
    bbox_part[blockIdx.x * 4 + 1] = mny;
    bbox_part[blockIdx.x * 4 + 2] = mxx;
    bbox_part[blockIdx.x * 4 + 3] = mxy;
  }
}

struct NodeParams {
  double min_x, min_y, res, r_a, r2, cell;
  int nx, ny, span, count;
};

// bbox -> clamped node window (center_select.cpp:36-50), single thread
__global__ void k_node_window(const double* __restrict__ part, int nparts, NodeParams p,
                              int* __restrict__ win) {
  double mnx = part[0], mny = part[1], mxx = part[2], mxy = part[3];
  for (int b = 1; b < nparts; ++b) {
    mnx = fmin(mnx, part[4 * b + 0]);
    mny = fmin(mny, part[4 * b + 1]);
    mxx = fmax(mxx, part[4 * b + 2]);
    mxy = fmax(mxy, part[4 * b + 3]);
  }
  // Rect::dilated (types.hpp:22-24)
  mnx = __dsub_rn(mnx, p.r_a);
  mny = __dsub_rn(mny, p.r_a);
  mxx = __dadd_rn(mxx, p.r_a);
  mxy = __dadd_rn(mxy, p.r_a);
  auto clamp_idx = [&](double v, double lo, int n) {
    const int i = static_cast<int>(floor(__dsub_rn(v, lo) / p.res));
    return min(max(i, 0), n);
  };
  win[0] = clamp_idx(mnx, p.min_x, p.nx);
  win[1] = clamp_idx(mxx, p.min_x, p.nx);
  win[2] = clamp_idx(mny, p.min_y, p.ny);
  win[3] = clamp_idx(mxy, p.min_y, p.ny);
}

__device__ __forceinline__ int lower_bound_u64(const uint64_t* __restrict__ a, int n, uint64_t k) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < k) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void k_count_nodes(const uint64_t* __restrict__ skey, const double* __restrict__ sx,
                              const double* __restrict__ sy, int m, NodeParams p,
                              const int* __restrict__ win, uint8_t* __restrict__ flag) {
  const int ny1 = p.ny + 1;
  const long long total = static_cast<long long>(p.nx + 1) * ny1;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = static_cast<int>(t / ny1), j = static_cast<int>(t % ny1);
    uint8_t ok = 0;
    if (i >= win[0] && i <= win[1] && j >= win[2] && j <= win[3]) {
      // node = roi.min + i * res (center_select.cpp:55-56), rounded twice
      const double nxp = __dadd_rn(p.min_x, __dmul_rn(static_cast<double>(i), p.res));
      const double nyp = __dadd_rn(p.min_y, __dmul_rn(static_cast<double>(j), p.res));
      const int cx = static_cast<int>(floor(nxp / p.cell));
      const int cy = static_cast<int>(floor(nyp / p.cell));
      int hits = 0;
      for (int ix = cx - p.span; ix <= cx + p.span && hits < p.count; ++ix)
        for (int iy = cy - p.span; iy <= cy + p.span && hits < p.count; ++iy) {
          const uint64_t k = cell_key(ix, iy);
          for (int q = lower_bound_u64(skey, m, k); q < m && __ldg(skey + q) == k; ++q) {
            const double d2 = sq2_exact(__ldg(sx + q) - nxp, __ldg(sy + q) - nyp);
            if (d2 <= p.r2 && ++hits >= p.count) break;
          }
        }
      ok = hits >= p.count;
    }
    flag[t] = ok;
  }
}

__global__ void k_gather_points(const uint32_t* __restrict__ idx, const double* __restrict__ x,
                                const double* __restrict__ y, int m, double* __restrict__ sx,
                                double* __restrict__ sy) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  sx[i] = x[idx[i]];
  sy[i] = y[idx[i]];
}

__global__ void k_node_coords(const int* __restrict__ sel, const int* __restrict__ nsel,
                              NodeParams p, double* __restrict__ ox, double* __restrict__ oy) {
  const int n = *nsel;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int lin = sel[t];
    const int i = lin / (p.ny + 1), j = lin % (p.ny + 1);
    ox[t] = __dadd_rn(p.min_x, __dmul_rn(static_cast<double>(i), p.res));
    oy[t] = __dadd_rn(p.min_y, __dmul_rn(static_cast<double>(j), p.res));
  }
}

size_t supported_nodes_device(tlg_ctx* ctx, const double* x, const double* y, size_t m,
                              const tlg_center_params& cp, const double** out_x,
                              const double** out_y) {
  cudaStream_t s = ctx->stream;
  require(m < (1ull << 31), TLG_INVALID_ARGUMENT, "too many observation points");
  NodeParams p;
  p.min_x = cp.roi_min_x;
  p.min_y = cp.roi_min_y;
  p.res = cp.mesh_resolution;
  p.r_a = cp.accept_radius;
  p.r2 = cp.accept_radius * cp.accept_radius;
  p.cell = std::max(cp.accept_radius, cp.mesh_resolution);  // center_select.cpp:27
  p.span = static_cast<int>(std::ceil(cp.accept_radius / p.cell));
  p.count = cp.accept_count;
  // center_select.cpp:31-34
  p.nx = static_cast<int>(std::floor((cp.roi_max_x - cp.roi_min_x) / cp.mesh_resolution + 1e-9));
  p.ny = static_cast<int>(std::floor((cp.roi_max_y - cp.roi_min_y) / cp.mesh_resolution + 1e-9));
  require(p.nx >= -1 && p.ny >= -1, TLG_INVALID_ARGUMENT, "degenerate roi");
  const long long total = static_cast<long long>(p.nx + 1) * (p.ny + 1);
  if (total <= 0) {
    *out_x = *out_y = nullptr;
    return 0;
  }
  require(total < (1ll << 31), TLG_INVALID_ARGUMENT, "mesh lattice too large");

  const int mi = static_cast<int>(m);
  uint64_t* key = ctx->ws<uint64_t>(S_KEYS, m);
  uint64_t* skey = ctx->ws<uint64_t>(S_KEYS2, m);
  uint32_t* idx = ctx->ws<uint32_t>(S_VALS, m);
  uint32_t* sidx = ctx->ws<uint32_t>(S_VALS2, m);
  const unsigned kb = static_cast<unsigned>(std::min<size_t>((m + 255) / 256, 2ull * ctx->num_sms));
  double* part = ctx->ws<double>(S_PARTIALS, 4 * kb);
  k_point_keys<<<kb, 256, 0, s>>>(x, y, m, p.cell, key, idx, part);
  TLG_LAUNCHED(ctx);
  int* win = ctx->ws<int>(S_COUNT, 8);
  k_node_window<<<1, 1, 0, s>>>(part, kb, p, win);
  TLG_LAUNCHED(ctx);
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, skey, idx, sidx, mi, 0, 64, s);
  void* dtmp = ctx->ws<unsigned char>(S_CUB, tmp);
  TLG_CUDA(cub::DeviceRadixSort::SortPairs(dtmp, tmp, key, skey, idx, sidx, mi, 0, 64, s));
  ++ctx->launches;
  double* sx = ctx->ws<double>(S_WORK1, m);
  double* sy = ctx->ws<double>(S_WORK2, m);
  k_gather_points<<<(mi + 255) / 256, 256, 0, s>>>(sidx, x, y, mi, sx, sy);
  TLG_LAUNCHED(ctx);

  uint8_t* flag = ctx->ws<uint8_t>(S_NODE_FLAG, static_cast<size_t>(total));
  const unsigned nb = static_cast<unsigned>(std::min<long long>((total + 255) / 256, 16ull * ctx->num_sms));
  k_count_nodes<<<nb, 256, 0, s>>>(skey, sx, sy, mi, p, win, flag);
  TLG_LAUNCHED(ctx);

  int* sel = ctx->ws<int>(S_NODE_IDX, static_cast<size_t>(total));
  int* nsel = win + 4;
  tmp = 0;
  thrust::counting_iterator<int> it(0);
  cub::DeviceSelect::Flagged(nullptr, tmp, it, flag, sel, nsel, static_cast<int>(total), s);
  dtmp = ctx->ws<unsigned char>(S_CUB, tmp);
  TLG_CUDA(cub::DeviceSelect::Flagged(dtmp, tmp, it, flag, sel, nsel, static_cast<int>(total), s));
  ++ctx->launches;
  int hn = 0;
  TLG_CUDA(cudaMemcpyAsync(&hn, nsel, sizeof(int), cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
  double* ox = ctx->ws<double>(S_NODES_X, static_cast<size_t>(hn) + 1);
  double* oy = ctx->ws<double>(S_NODES_Y, static_cast<size_t>(hn) + 1);
  if (hn > 0) {
    k_node_coords<<<(hn + 255) / 256, 256, 0, s>>>(sel, nsel, p, ox, oy);
    TLG_LAUNCHED(ctx);
  }
  *out_x = ox;
  *out_y = oy;
  return static_cast<size_t>(hn);
}

}  // namespace tlg
