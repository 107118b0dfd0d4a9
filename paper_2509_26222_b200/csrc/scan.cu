// Per-scan spatial binning of lever arms (tlg_scan_*).
//
// lm_solve re-evaluates the same scan's manifold rows every LM iteration
// (scan_matcher.cpp:276,315) under poses that differ by centimetres. Binning
// the lever arms once per scan by the lattice cell (or centre-grid cell)
// their world position falls in under the scan's initial pose makes the
// 32 points of a warp share one node window, so weight-grid reads become
// warp-broadcast hits instead of 32 scattered gathers. Correctness never
// depends on the binning: a point that drifts to another cell is simply
// evaluated with its own window.
#include <cub/cub.cuh>

#include "internal.cuh"

namespace tlg {

struct BinParams {
  double R[9], t[3];
  double org_x, org_y, inv_cell;
  int nx, ny;
  int sub;  // sub-cells per axis inside a cell (power of two), 1 = none
};

__global__ void k_bin_keys(BinParams p, const double* __restrict__ hx, const double* __restrict__ hy,
                           const double* __restrict__ hz, size_t n, uint32_t* __restrict__ key,
                           uint32_t* __restrict__ idx) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double h0 = hx[i], h1 = hy[i], h2 = hz[i];
  const double x = p.R[0] * h0 + p.R[1] * h1 + p.R[2] * h2 + p.t[0];
  const double y = p.R[3] * h0 + p.R[4] * h1 + p.R[5] * h2 + p.t[1];
  double fx = (x - p.org_x) * p.inv_cell, fy = (y - p.org_y) * p.inv_cell;
  fx = isfinite(fx) ? fmin(fmax(fx, 0.0), p.nx - 1.0) : 0.0;
  fy = isfinite(fy) ? fmin(fmax(fy, 0.0), p.ny - 1.0) : 0.0;
  // cell-major, then a sub-cell (row-major p.sub x p.sub) inside the cell:
  // a warp's run of points stays compact, so a small pose change between
  // binning and evaluation moves it into few distinct lattice windows
  const uint32_t cx = static_cast<uint32_t>(fx), cy = static_cast<uint32_t>(fy);
  const uint32_t sx = min(static_cast<uint32_t>((fx - cx) * p.sub), static_cast<uint32_t>(p.sub - 1));
  const uint32_t sy = min(static_cast<uint32_t>((fy - cy) * p.sub), static_cast<uint32_t>(p.sub - 1));
  key[i] = (cx * static_cast<uint32_t>(p.ny) + cy) * static_cast<uint32_t>(p.sub * p.sub) +
           sx * static_cast<uint32_t>(p.sub) + sy;
  idx[i] = static_cast<uint32_t>(i);
}

__global__ void k_bin_gather(const uint32_t* __restrict__ perm, size_t n,
                             const double* __restrict__ hx, const double* __restrict__ hy,
                             const double* __restrict__ hz, double* __restrict__ ox,
                             double* __restrict__ oy, double* __restrict__ oz) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t j = perm[i];
  ox[i] = hx[j];
  oy[i] = hy[j];
  oz[i] = hz[j];
}

tlg_scan* scan_create(tlg_model* m, const double R0[9], const double t0[3], const double* hx,
                      const double* hy, const double* hz, size_t n) {
  tlg_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  ensure_grid(m);
  require(n < (1ull << 32), TLG_INVALID_ARGUMENT, "scan too large");
  auto* sc = new tlg_scan();
  try {
    sc->ctx = ctx;
    sc->n = n;
    sc->hx.ensure(n);
    sc->hy.ensure(n);
    sc->hz.ensure(n);
    sc->perm.ensure(n);
    if (n == 0) return sc;
    BinParams p;
    for (int i = 0; i < 9; ++i) p.R[i] = R0[i];
    for (int i = 0; i < 3; ++i) p.t[i] = t0[i];
    if (m->lat.valid) {
      p.org_x = m->lat.org_x;
      p.org_y = m->lat.org_y;
      p.inv_cell = m->lat.inv_res;
      p.nx = m->lat.ni;
      p.ny = m->lat.nj;
    } else {
      const CenterGrid& g = m->grid;
      p.org_x = g.gx0 * g.cell;
      p.org_y = g.gy0 * g.cell;
      p.inv_cell = 1.0 / g.cell;
      p.nx = std::max(1, g.gnx);
      p.ny = std::max(1, g.gny);
    }
    cudaEvent_t e0, e1;
    TLG_CUDA(cudaEventCreate(&e0));
    TLG_CUDA(cudaEventCreate(&e1));
    TLG_CUDA(cudaEventRecord(e0, s));
    uint32_t* key = ctx->ws<uint32_t>(S_KEYS, n);
    uint32_t* key2 = ctx->ws<uint32_t>(S_KEYS2, n);
    uint32_t* idx = ctx->ws<uint32_t>(S_VALS, n);
    const unsigned long long cells = static_cast<unsigned long long>(p.nx) * p.ny;
    p.sub = cells * 16 <= (1ull << 32) ? 4 : (cells * 4 <= (1ull << 32) ? 2 : 1);
    k_bin_keys<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, hx, hy, hz, n, key, idx);
    TLG_LAUNCHED(ctx);
    int end_bit = 1;
    const unsigned long long keys = cells * p.sub * p.sub;
    while (end_bit < 32 && (1ull << end_bit) < keys) ++end_bit;
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, key2, idx, sc->perm.p, (int)n, 0, end_bit, s);
    void* dtmp = ctx->ws<unsigned char>(S_CUB, tmp);
    TLG_CUDA(cub::DeviceRadixSort::SortPairs(dtmp, tmp, key, key2, idx, sc->perm.p, (int)n, 0,
                                             end_bit, s));
    ++ctx->launches;
    k_bin_gather<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(sc->perm.p, n, hx, hy, hz, sc->hx.p,
                                                            sc->hy.p, sc->hz.p);
    TLG_LAUNCHED(ctx);
    TLG_CUDA(cudaEventRecord(e1, s));
    TLG_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    TLG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    sc->bin_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return sc;
  } catch (...) {
    delete sc;
    throw;
  }
}

}  // namespace tlg
