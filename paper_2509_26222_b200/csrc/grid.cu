// K1 centre_hash_build: GridIndex2 (grid_index.hpp:16-66) over the model's
// centres as a dense CSR cell array in HBM. Cell coordinates use the
// reference's exact expression static_cast<int>(floor(v / cell)); ids stay
// ascending inside each cell (stable radix sort), and centre coordinates
// and weights are stored in cell order so a 3x3 cell sweep reads contiguous
// runs.
#include <cub/cub.cuh>

#include <climits>
#include <cmath>

#include "internal.cuh"

namespace tlg {

__global__ void k_cell_coords(const double* __restrict__ cx, const double* __restrict__ cy,
                              size_t n, double cell, int* __restrict__ ix, int* __restrict__ iy,
                              int* __restrict__ bbox) {
  int mnx = INT_MAX, mny = INT_MAX, mxx = INT_MIN, mxy = INT_MIN;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const int a = static_cast<int>(floor(cx[i] / cell));
    const int b = static_cast<int>(floor(cy[i] / cell));
    ix[i] = a;
    iy[i] = b;
    mnx = min(mnx, a);
    mny = min(mny, b);
    mxx = max(mxx, a);
    mxy = max(mxy, b);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mnx = min(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
    mny = min(mny, __shfl_xor_sync(0xffffffffu, mny, o));
    mxx = max(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
    mxy = max(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&bbox[0], mnx);
    atomicMin(&bbox[1], mny);
    atomicMax(&bbox[2], mxx);
    atomicMax(&bbox[3], mxy);
  }
}

__global__ void k_cell_linear(const int* __restrict__ ix, const int* __restrict__ iy, size_t n,
                              int gx0, int gy0, int gny, uint32_t* __restrict__ key,
                              uint32_t* __restrict__ id, int* __restrict__ counts) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t k = static_cast<uint32_t>(ix[i] - gx0) * static_cast<uint32_t>(gny) +
                     static_cast<uint32_t>(iy[i] - gy0);
  key[i] = k;
  id[i] = static_cast<uint32_t>(i);
  atomicAdd(&counts[k], 1);
}

__global__ void k_gather_sorted(const uint32_t* __restrict__ sid, size_t n,
                                const double* __restrict__ cx, const double* __restrict__ cy,
                                const double* __restrict__ w, double* __restrict__ scx,
                                double* __restrict__ scy, double* __restrict__ sw) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t j = sid[i];
  if (scx) scx[i] = cx[j];
  if (scy) scy[i] = cy[j];
  sw[i] = w[j];
}

void build_center_grid(tlg_model* m) {
  tlg_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  CenterGrid& g = m->grid;
  const size_t n = m->hcx.size();
  g.cell = std::min(m->kernel.cutoff_radius, 1e6);  // terrain_model.cpp:63
  g.span = static_cast<int>(std::ceil(m->kernel.cutoff_radius / g.cell));
  if (n == 0) {
    g.gx0 = g.gy0 = 0;
    g.gnx = g.gny = 0;
    g.cell_start.ensure(2);
    TLG_CUDA(cudaMemsetAsync(g.cell_start.p, 0, 2 * sizeof(int), s));
    m->grid_dirty = false;
    return;
  }
  int* ix = ctx->ws<int>(S_KEYS, n);
  int* iy = ctx->ws<int>(S_KEYS2, n);
  int* bbox = ctx->ws<int>(S_COUNT, 4);
  const int hb[4] = {INT_MAX, INT_MAX, INT_MIN, INT_MIN};
  TLG_CUDA(cudaMemcpyAsync(bbox, hb, sizeof(hb), cudaMemcpyHostToDevice, s));
  const unsigned blocks = static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 4 * 148));
  k_cell_coords<<<blocks, 256, 0, s>>>(m->cx.p, m->cy.p, n, g.cell, ix, iy, bbox);
  TLG_LAUNCHED(ctx);
  int hbox[4];
  TLG_CUDA(cudaMemcpyAsync(hbox, bbox, sizeof(hbox), cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
  g.gx0 = hbox[0];
  g.gy0 = hbox[1];
  const long long gnx = static_cast<long long>(hbox[2]) - hbox[0] + 1;
  const long long gny = static_cast<long long>(hbox[3]) - hbox[1] + 1;
  require(gnx * gny <= (1ll << 27), TLG_RUNTIME_ERROR,
          "centre spread too large for the dense centre grid");
  g.gnx = static_cast<int>(gnx);
  g.gny = static_cast<int>(gny);
  const size_t ncell = static_cast<size_t>(gnx * gny);

  g.cell_start.ensure(ncell + 1);
  TLG_CUDA(cudaMemsetAsync(g.cell_start.p, 0, (ncell + 1) * sizeof(int), s));
  uint32_t* key = ctx->ws<uint32_t>(S_VALS, n);
  uint32_t* key2 = ctx->ws<uint32_t>(S_VALS2, n);
  uint32_t* id = ctx->ws<uint32_t>(S_NODE_IDX, n);
  g.sorted_id.ensure(n);
  k_cell_linear<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ix, iy, n, g.gx0, g.gy0, g.gny, key,
                                                           id, g.cell_start.p);
  TLG_LAUNCHED(ctx);
  // stable radix sort by cell -> ids ascending within a cell
  int end_bit = 1;
  while (end_bit < 32 && (1ull << end_bit) < ncell) ++end_bit;
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, key2, id, g.sorted_id.p, (int)n, 0, end_bit, s);
  void* dtmp = ctx->ws<unsigned char>(S_CUB, tmp);
  TLG_CUDA(cub::DeviceRadixSort::SortPairs(dtmp, tmp, key, key2, id, g.sorted_id.p, (int)n, 0,
                                           end_bit, s));
  ++ctx->launches;
  // counts -> exclusive starts (in place over ncell+1 entries)
  tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, g.cell_start.p, g.cell_start.p, (int)(ncell + 1), s);
  dtmp = ctx->ws<unsigned char>(S_CUB, tmp);
  TLG_CUDA(cub::DeviceScan::ExclusiveSum(dtmp, tmp, g.cell_start.p, g.cell_start.p,
                                         (int)(ncell + 1), s));
  ++ctx->launches;
  g.scx.ensure(n);
  g.scy.ensure(n);
  g.sw.ensure(n);
  k_gather_sorted<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g.sorted_id.p, n, m->cx.p, m->cy.p,
                                                             m->w.p, g.scx.p, g.scy.p, g.sw.p);
  TLG_LAUNCHED(ctx);
  m->grid_dirty = false;
}

void ensure_grid(tlg_model* m) {
  if (m->grid_dirty) build_center_grid(m);
}

void sync_weights_to_grid(tlg_model* m) {
  if (m->grid_dirty) {
    build_center_grid(m);
    return;
  }
  const size_t n = m->hcx.size();
  if (n == 0) return;
  k_gather_sorted<<<(unsigned)((n + 255) / 256), 256, 0, m->ctx->stream>>>(
      m->grid.sorted_id.p, n, m->cx.p, m->cy.p, m->w.p, nullptr, nullptr, m->grid.sw.p);
  TLG_LAUNCHED(m->ctx);
}

GridView grid_view(const tlg_model* m) {
  const CenterGrid& g = m->grid;
  return GridView{g.scx.p, g.scy.p, g.sw.p, g.sorted_id.p, g.cell_start.p, g.cell,
                  g.span,  g.gx0,   g.gy0,  g.gnx,         g.gny};
}

}  // namespace tlg
