// Model state: host-side structure mirror (terrain_model.cpp:26-95) and the
// device-resident numeric state (centres, weights, block info_inv pool).
#include <cmath>

#include "internal.cuh"

namespace tlg {

void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  std::string msg = std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                    std::to_string(line) + ")";
  throw Error(e == cudaErrorMemoryAllocation ? TLG_OUT_OF_MEMORY : TLG_CUDA_ERROR, msg);
}

// kernel.cpp:15-25
void finalize_kernel(tlg_kernel_params& k) {
  if (!(k.sigma > 0.0)) throw Error(TLG_INVALID_ARGUMENT, "kernel sigma must be > 0");
  if (k.sigma_eps < 0.0) throw Error(TLG_INVALID_ARGUMENT, "sigma_eps must be >= 0");
  if (!(k.lambda > 0.0)) throw Error(TLG_INVALID_ARGUMENT, "lambda must be > 0");
  const double st = std::sqrt(k.sigma * k.sigma + k.sigma_eps * k.sigma_eps);
  k.cutoff_radius = std::max(k.cutoff_radius, 3.0 * st);
  if (!std::isfinite(k.sigma) || !std::isfinite(k.sigma_eps) || !std::isfinite(k.lambda))
    throw Error(TLG_INVALID_ARGUMENT, "non-finite kernel parameter");
}

KernelConst make_kernel_const(const tlg_kernel_params& k) {
  KernelConst c;
  c.sigma = k.sigma;
  c.sigma_eps = k.sigma_eps;
  c.lambda = k.lambda;
  c.cutoff = k.cutoff_radius;
  c.r2 = k.cutoff_radius * k.cutoff_radius;
  c.neg_inv_2s2 = -1.0 / (2.0 * k.sigma * k.sigma);
  c.sigma_tilde = std::sqrt(k.sigma * k.sigma + k.sigma_eps * k.sigma_eps);
  c.neg_inv_2st2 = -1.0 / (2.0 * c.sigma_tilde * c.sigma_tilde);
  c.inv_s2 = 1.0 / (k.sigma * k.sigma);
  const double st2 = k.sigma * k.sigma + k.sigma_eps * k.sigma_eps;
  c.scale = k.sigma * k.sigma / st2;
  return c;
}

// terrain_model.cpp:15-22
int64_t pack2(int64_t x, int64_t y) {
  return static_cast<int64_t>((static_cast<uint64_t>(x) << 32)) ^ (y & 0xffffffffll);
}

// terrain_model.cpp:46-51
int64_t tile_key(const tlg_model* m, double cx, double cy) {
  const double side = 2.0 * m->kernel.cutoff_radius;
  if (!(side < 1e12)) return 0;
  return pack2(static_cast<int64_t>(std::floor(cx / side)),
               static_cast<int64_t>(std::floor(cy / side)));
}

int64_t mesh_node_key(const tlg_model* m, double x, double y) {
  const double res = m->cparams.mesh_resolution;
  return pack2(std::llround((x - m->cparams.roi_min_x) / res),
               std::llround((y - m->cparams.roi_min_y) / res));
}

// terrain_model.cpp:53-60
uint32_t block_for_tile(tlg_model* m, int64_t key) {
  auto it = m->tile_blocks.find(key);
  if (it != m->tile_blocks.end()) return it->second;
  const auto id = static_cast<uint32_t>(m->members.size());
  m->tile_blocks.emplace(key, id);
  m->members.emplace_back();
  m->blk_off.push_back(0);
  m->blk_ld.push_back(0);
  return id;
}

static inline int round_up8(int v) { return (v + 7) & ~7; }

__global__ void k_copy_block(const double* __restrict__ src, int sld, double* __restrict__ dst,
                             int dld, int n) {
  for (int c = blockIdx.x; c < n; c += gridDim.x)
    for (int r = threadIdx.x; r < n; r += blockDim.x) dst[(size_t)c * dld + r] = src[(size_t)c * sld + r];
}

// New rows/cols [old_n, new_n) of a block: zero couplings, diagonal 1/lambda
// (terrain_model.cpp:84-88).
__global__ void k_grow_block(double* __restrict__ a, int ld, int old_n, int new_n, double diag) {
  for (int c = blockIdx.x; c < new_n; c += gridDim.x)
    for (int r = threadIdx.x; r < new_n; r += blockDim.x)
      if (r >= old_n || c >= old_n) a[(size_t)c * ld + r] = (r == c) ? diag : 0.0;
}

__global__ void k_set_diag(double* __restrict__ pool, const size_t* __restrict__ pos, size_t n,
                           double v) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i < n) pool[pos[i]] = v;
}

// Ensure block b has room for new_size and initialise the grown rows/cols.
// old size = current blk "size" recorded in ld bookkeeping via members before
// the append: caller passes old_n.
static void repack_pool(tlg_model* m, size_t extra) {
  tlg_ctx* ctx = m->ctx;
  size_t need = extra;
  for (size_t b = 0; b < m->members.size(); ++b)
    need += static_cast<size_t>(m->blk_ld[b]) * m->blk_ld[b];
  DBuf<double> np;
  np.ensure(need + 64);
  size_t off = 0;
  for (size_t b = 0; b < m->members.size(); ++b) {
    const int ld = m->blk_ld[b];
    if (ld > 0 && m->pool.p) {
      TLG_CUDA(cudaMemcpyAsync(np.p + off, m->pool.p + m->blk_off[b],
                               sizeof(double) * ld * ld, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    m->blk_off[b] = off;
    off += static_cast<size_t>(ld) * ld;
  }
  TLG_CUDA(cudaStreamSynchronize(ctx->stream));
  m->pool = std::move(np);
  m->pool_used = off;
}

void block_resize(tlg_model* m, uint32_t b, int old_n, int new_n) {
  tlg_ctx* ctx = m->ctx;
  int ld = m->blk_ld[b];
  if (new_n > ld) {
    const int nld = round_up8(std::max(new_n, ld + ld / 2));
    const size_t sz = static_cast<size_t>(nld) * nld;
    if (m->pool_used + sz > m->pool.n) {
      // compact live blocks and leave headroom
      repack_pool(m, sz + (m->pool_used + sz) / 2);
    }
    const size_t noff = m->pool_used;
    if (old_n > 0) {
      k_copy_block<<<std::min(old_n, 1024), 128, 0, ctx->stream>>>(m->pool.p + m->blk_off[b], ld,
                                                                   m->pool.p + noff, nld, old_n);
      TLG_LAUNCHED(ctx);
    }
    m->blk_off[b] = noff;
    m->blk_ld[b] = nld;
    m->pool_used += sz;
    ld = nld;
  }
  if (new_n > old_n) {
    k_grow_block<<<std::min(new_n, 1024), 128, 0, ctx->stream>>>(
        m->pool.p + m->blk_off[b], ld, old_n, new_n, 1.0 / m->kernel.lambda);
    TLG_LAUNCHED(ctx);
  }
}

void ensure_dev_capacity(tlg_model* m, size_t n) {
  if (n <= m->dev_cap && m->cx.p) return;
  const size_t keep = std::min(m->dev_cap, m->hcx.size());
  const size_t cap = std::max<size_t>(n + n / 2, 64);
  cudaStream_t s = m->ctx->stream;
  m->cx.grow_keep(cap, keep, s);
  m->cy.grow_keep(cap, keep, s);
  m->w.grow_keep(cap, keep, s);
  m->d_block_index.grow_keep(cap, keep, s);
  m->dev_cap = cap;
}

// Append centres (host mirror already updated for ids [first, n)); uploads
// coordinates, zero weights, block ids.
void upload_new_centres(tlg_model* m, size_t first) {
  const size_t n = m->hcx.size();
  if (n == first) return;
  ensure_dev_capacity(m, n);
  tlg_ctx* ctx = m->ctx;
  const size_t k = n - first;
  TLG_CUDA(cudaMemcpyAsync(m->cx.p + first, m->hcx.data() + first, k * 8, cudaMemcpyHostToDevice, ctx->stream));
  TLG_CUDA(cudaMemcpyAsync(m->cy.p + first, m->hcy.data() + first, k * 8, cudaMemcpyHostToDevice, ctx->stream));
  TLG_CUDA(cudaMemsetAsync(m->w.p + first, 0, k * 8, ctx->stream));
  TLG_CUDA(cudaMemcpyAsync(m->d_block_index.p + first, m->block_index.data() + first, k * 4,
                           cudaMemcpyHostToDevice, ctx->stream));
  // pageable sources: make sure the copies completed before the vectors move
  TLG_CUDA(cudaStreamSynchronize(ctx->stream));
  m->grid_dirty = true;
}

// terrain_model.cpp:77-95 (host bookkeeping part of add_center). Returns
// the block id; device-side growth is batched by the caller.
uint32_t add_center_host(tlg_model* m, double x, double y) {
  const auto id = static_cast<uint32_t>(m->hcx.size());
  m->hcx.push_back(x);
  m->hcy.push_back(y);
  const uint32_t b = block_for_tile(m, tile_key(m, x, y));
  m->block_index.push_back(b);
  m->members[b].push_back(id);
  m->occupancy.insert(mesh_node_key(m, x, y));
  return id;
}

}  // namespace tlg

using namespace tlg;

// terrain_model.cpp:26-44
tlg_model* model_create_impl(tlg_ctx* ctx, const tlg_kernel_params& k0,
                             const tlg_center_params& cp, const double* hx, const double* hy,
                             size_t n) {
  auto* m = new tlg_model();
  try {
    m->ctx = ctx;
    m->kernel = k0;
    finalize_kernel(m->kernel);
    m->kc = make_kernel_const(m->kernel);
    m->cparams = cp;
    m->hcx.reserve(n);
    m->hcy.reserve(n);
    for (size_t i = 0; i < n; ++i) {
      m->hcx.push_back(hx[i]);
      m->hcy.push_back(hy[i]);
      const uint32_t b = block_for_tile(m, tile_key(m, hx[i], hy[i]));
      m->block_index.push_back(b);
      m->members[b].push_back(static_cast<uint32_t>(i));
    }
    // rebuild_indexes (terrain_model.cpp:62-70): mesh occupancy
    for (size_t i = 0; i < n; ++i) m->occupancy.insert(mesh_node_key(m, hx[i], hy[i]));
    // info_inv = I / lambda per block
    size_t total = 0;
    for (size_t b = 0; b < m->members.size(); ++b) {
      const int ld = std::max(8, (static_cast<int>(m->members[b].size()) + 7) & ~7);
      m->blk_ld[b] = ld;
      m->blk_off[b] = total;
      total += static_cast<size_t>(ld) * ld;
    }
    m->pool.ensure(total + total / 2 + 64);
    m->pool_used = total;
    TLG_CUDA(cudaMemsetAsync(m->pool.p, 0, sizeof(double) * total, ctx->stream));
    if (n > 0) {
      std::vector<size_t> pos(n);
      std::vector<int> local(m->members.size(), 0);
      for (size_t i = 0; i < n; ++i) {
        const uint32_t b = m->block_index[i];
        const size_t k = static_cast<size_t>(local[b]++);
        pos[i] = m->blk_off[b] + k * m->blk_ld[b] + k;
      }
      size_t* dpos = ctx->ws<size_t>(S_WORK1, n);
      TLG_CUDA(cudaMemcpyAsync(dpos, pos.data(), n * sizeof(size_t), cudaMemcpyHostToDevice, ctx->stream));
      k_set_diag<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(m->pool.p, dpos, n, 1.0 / m->kernel.lambda);
      TLG_LAUNCHED(ctx);
      TLG_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    upload_new_centres(m, 0);
    build_center_grid(m);
    return m;
  } catch (...) {
    delete m;
    throw;
  }
}
