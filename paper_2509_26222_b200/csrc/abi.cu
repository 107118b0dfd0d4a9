// extern "C" entry points of include/terralio_gpu.h. Each one converts
// internal exceptions into the status enum + a thread-local message.
#include <cub/cub.cuh>
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>

#include "internal.cuh"

using namespace tlg;

tlg_model* model_create_impl(tlg_ctx* ctx, const tlg_kernel_params& k0,
                             const tlg_center_params& cp, const double* hx, const double* hy,
                             size_t n);
namespace tlg {
void block_resize(tlg_model* m, uint32_t b, int old_n, int new_n);
void upload_new_centres(tlg_model* m, size_t first);
uint32_t add_center_host(tlg_model* m, double x, double y);
void moment_device(tlg_model* m, const double* x, const double* y, size_t n, uint32_t* rowp,
                   uint32_t** ids, double** vals, size_t* nnz);
void manifold_device_streamed(tlg_model* m, const double R[9], const double t[3],
                              const double* hx, const double* hy, const double* hz, size_t n,
                              double wheel_radius, double lambda_M, double huber, double* r,
                              double* J, uint8_t* valid, double* raw, tlg_normal_eq* ne);
size_t select_ground_device(tlg_ctx* ctx, const double* px, const double* py, const double* pz,
                            const uint8_t* kind, size_t n, const double R[9], const double t[3],
                            const double roi[4], double radius, double voxel, size_t max_points,
                            double* ox, double* oy, double* oz);
void map_insert(tlg_map* m, const double* px, const double* py, const double* pz,
                const uint8_t* kind, const int* label, size_t n, const double R[9],
                const double t[3]);
size_t build_correspondences_device(tlg_map* m, const double* px, const double* py,
                                    const double* pz, const uint8_t* kind, size_t n,
                                    const double R[9], const double t[3], const double cfgv[11]);
void feature_rows_device(tlg_ctx* ctx, size_t nc, const int32_t* kind, const double* ps,
                         const double* par, const double* wgt, const double R[9], const double t[3],
                         double* r, double* J, size_t* rows_out);
void feature_normal_eq_device(tlg_map* m, const double R[9], const double t[3], double ne29[29]);
tlg_map* map_new(tlg_ctx* ctx, double voxel, size_t window);
void map_free(tlg_map* m);
size_t map_points_host(tlg_map* m, int kind, double* xyz, int32_t* labels, size_t cap);
tlg_ctx* map_ctx(tlg_map* m);
bool lm_step_device(tlg_ctx* ctx, const double ne29[29], double mu, double delta[6]);
double eigmin6_device(tlg_ctx* ctx, const double ne29[29]);
size_t correspondences_host(tlg_map* m, int32_t* kind, uint32_t* feature, double* params,
                            double* weight, int32_t* label, double* dist, double* fitq,
                            size_t cap);
void error_histogram_device(tlg_model* m, const double* x, const double* y, const double* z,
                            size_t n, double trim_fraction, int bins, double* edges,
                            uint64_t* counts, uint64_t* trimmed, uint64_t* overflow);
tlg_scan* scan_create(tlg_model* m, const double R0[9], const double t0[3], const double* hx,
                      const double* hy, const double* hz, size_t n);
}  // namespace tlg

namespace {
thread_local std::string g_err;

template <typename F>
tlg_status guard(F&& f) {
  try {
    f();
    return TLG_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return TLG_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_err = e.what();
    return TLG_RUNTIME_ERROR;
  }
}

void check_ptr(const void* p, const char* what) {
  if (!p) throw Error(TLG_INVALID_ARGUMENT, std::string("null argument: ") + what);
}
}  // namespace

// Pinned staging buffer; the stream is drained first so a previous async
// copy out of the buffer can never be overwritten.
void* tlg_ctx::host_stage(size_t bytes) {
  TLG_CUDA(cudaStreamSynchronize(stream));
  if (bytes > pinned_bytes) {
    // pinned allocations cost milliseconds: grow with headroom (per-scan
    // table sizes creep up with the active set), at least 1 MiB
    const size_t cap = std::max(bytes + bytes / 2, size_t{1} << 20);
    if (pinned) cudaFreeHost(pinned);
    pinned = nullptr;
    pinned_bytes = 0;
    TLG_CUDA(cudaMallocHost(&pinned, cap));
    pinned_bytes = cap;
  }
  return pinned;
}

void tlg_ctx::sync() { TLG_CUDA(cudaStreamSynchronize(stream)); }

namespace tlg {
void copy_in(tlg_ctx* ctx, void* dst, const void* src, size_t bytes, tlg_mem mem) {
  if (!bytes) return;
  TLG_CUDA(cudaMemcpyAsync(dst, src, bytes,
                           mem == TLG_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                           ctx->stream));
}
void copy_out(tlg_ctx* ctx, void* dst, const void* src, size_t bytes, tlg_mem mem) {
  if (!bytes) return;
  TLG_CUDA(cudaMemcpyAsync(dst, src, bytes,
                           mem == TLG_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                           ctx->stream));
}
}  // namespace tlg

extern "C" {

int tlg_abi_version(void) { return TLG_ABI_VERSION; }
const char* tlg_last_error(void) { return g_err.c_str(); }

tlg_status tlg_ctx_create(int device, void* stream, tlg_ctx** out) {
  return guard([&] {
    check_ptr(out, "out");
    int ndev = 0;
    TLG_CUDA(cudaGetDeviceCount(&ndev));
    require(device >= 0 && device < ndev, TLG_INVALID_ARGUMENT, "bad device ordinal");
    cudaDeviceProp prop;
    TLG_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      throw Error(TLG_CUDA_ERROR, "terralio_gpu is built for sm_100a (B200); device is sm_" +
                                      std::to_string(prop.major) + std::to_string(prop.minor));
    TLG_CUDA(cudaSetDevice(device));
    auto* c = new tlg_ctx();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    // NULL is the legacy default stream (torch's default stream), not a
    // private one: device inputs written by the caller on that stream are
    // then ordered before the library's reads without an extra event.
    c->stream = static_cast<cudaStream_t>(stream);
    *out = c;
  });
}

tlg_status tlg_ctx_destroy(tlg_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    cudaStreamSynchronize(ctx->stream);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->copy_stream) {
      cudaStreamSynchronize(ctx->copy_stream);
      for (auto& e : ctx->copy_ev)
        if (e) cudaEventDestroy(e);
      cudaStreamDestroy(ctx->copy_stream);
    }
    delete ctx;
  });
}

tlg_status tlg_ctx_set_stream(tlg_ctx* ctx, void* stream) {
  return guard([&] {
    check_ptr(ctx, "ctx");
    ctx->sync();
    ctx->stream = static_cast<cudaStream_t>(stream);
  });
}

tlg_status tlg_ctx_synchronize(tlg_ctx* ctx) {
  return guard([&] {
    check_ptr(ctx, "ctx");
    ctx->sync();
  });
}

uint64_t tlg_ctx_launch_count(const tlg_ctx* ctx) { return ctx ? ctx->launches : 0; }

tlg_status tlg_ctx_set_profiling(tlg_ctx* ctx, int enable) {
  return guard([&] {
    check_ptr(ctx, "ctx");
    ctx->profiling = enable != 0;
    for (int i = 0; i < 4; ++i) {
      ctx->prof_ms[i] = 0.0;
      ctx->prof_n[i] = 0;
    }
  });
}

tlg_status tlg_ctx_kernel_stats(tlg_ctx* ctx, int kernel, double* total_ms, uint64_t* launches) {
  return guard([&] {
    check_ptr(ctx, "ctx");
    require(kernel >= 0 && kernel < 4, TLG_INVALID_ARGUMENT, "bad kernel id");
    if (total_ms) *total_ms = ctx->prof_ms[kernel];
    if (launches) *launches = ctx->prof_n[kernel];
  });
}

tlg_status tlg_select_ground_points(tlg_ctx* ctx, const double* px, const double* py,
                                    const double* pz, const uint8_t* kind, size_t n,
                                    tlg_mem in_mem, const double R[9], const double t[3],
                                    const double roi_min[2], const double roi_max[2],
                                    double ground_radius, double ground_voxel,
                                    size_t max_points, double* out_x, double* out_y,
                                    double* out_z, tlg_mem out_mem, size_t* out_n) {
  return guard([&] {
    check_ptr(ctx, "ctx");
    check_ptr(R, "R");
    check_ptr(t, "t");
    check_ptr(roi_min, "roi_min");
    check_ptr(roi_max, "roi_max");
    check_ptr(out_n, "out_n");
    require(ground_voxel > 0.0, TLG_INVALID_ARGUMENT, "ground_voxel must be positive");
    *out_n = 0;
    if (n == 0 || max_points == 0) return;
    const double* dx = as_device(ctx, S_IN_HX, px, n, in_mem);
    const double* dy = as_device(ctx, S_IN_HY, py, n, in_mem);
    const double* dz = as_device(ctx, S_IN_HZ, pz, n, in_mem);
    const uint8_t* dk = as_device(ctx, S_MOMENT_ROW, kind, n, in_mem);
    const bool dev = out_mem == TLG_DEVICE;
    double* ox = out_x ? (dev ? out_x : ctx->ws<double>(S_OUT_R, max_points)) : nullptr;
    double* oy = out_y ? (dev ? out_y : ctx->ws<double>(S_OUT_GX, max_points)) : nullptr;
    double* oz = out_z ? (dev ? out_z : ctx->ws<double>(S_OUT_GY, max_points)) : nullptr;
    const double roi[4] = {roi_min[0], roi_min[1], roi_max[0], roi_max[1]};
    const size_t k = select_ground_device(ctx, dx, dy, dz, dk, n, R, t, roi, ground_radius,
                                          ground_voxel, max_points, ox, oy, oz);
    if (!dev && k) {
      if (out_x) copy_out(ctx, out_x, ox, k * 8, TLG_HOST);
      if (out_y) copy_out(ctx, out_y, oy, k * 8, TLG_HOST);
      if (out_z) copy_out(ctx, out_z, oz, k * 8, TLG_HOST);
    }
    ctx->sync();
    *out_n = k;
  });
}

tlg_status tlg_terrain_error_histogram(tlg_model* m, const double* x, const double* y,
                                       const double* z, size_t n, tlg_mem mem,
                                       double trim_fraction, int bins, double* edges,
                                       uint64_t* counts, uint64_t* trimmed, uint64_t* overflow) {
  return guard([&] {
    check_ptr(m, "model");
    check_ptr(edges, "edges");
    check_ptr(counts, "counts");
    check_ptr(trimmed, "trimmed");
    check_ptr(overflow, "overflow");
    require(n > 0 && x && y && z, TLG_INVALID_ARGUMENT, "histogram needs matched non-empty samples");
    tlg_ctx* ctx = m->ctx;
    const double* dx = as_device(ctx, S_IN_X, x, n, mem);
    const double* dy = as_device(ctx, S_IN_Y, y, n, mem);
    const double* dz = as_device(ctx, S_IN_Z, z, n, mem);
    error_histogram_device(m, dx, dy, dz, n, trim_fraction, bins, edges, counts, trimmed,
                           overflow);
  });
}

tlg_status tlg_lm_step(tlg_ctx* ctx, const tlg_normal_eq* ne, double mu, double delta[6]) {
  return guard([&] {
    check_ptr(ctx, "ctx");
    check_ptr(ne, "ne");
    check_ptr(delta, "delta");
    double v[29];
    for (int k = 0; k < 21; ++k) v[k] = ne->A[k];
    for (int k = 0; k < 6; ++k) v[21 + k] = ne->g[k];
    v[27] = ne->cost;
    v[28] = ne->valid;
    if (!lm_step_device(ctx, v, mu, delta)) throw Error(TLG_RUNTIME_ERROR, "non-finite LM step");
  });
}

tlg_status tlg_ne_min_eigenvalue(tlg_ctx* ctx, const tlg_normal_eq* ne, double* lambda_min) {
  return guard([&] {
    check_ptr(ctx, "ctx");
    check_ptr(ne, "ne");
    check_ptr(lambda_min, "lambda_min");
    double v[29] = {0};
    for (int k = 0; k < 21; ++k) v[k] = ne->A[k];
    *lambda_min = eigmin6_device(ctx, v);
  });
}

tlg_status tlg_match_config_default(tlg_match_config* c) {
  return guard([&] {
    check_ptr(c, "cfg");
    *c = tlg_match_config{1.0, 0.1, 0.025, 5.0, 3.0, 0.05, 0.05, 5.0, 0.003, 0.25, 4.0};
  });
}

tlg_status tlg_map_create(tlg_ctx* ctx, double voxel_size, size_t window, tlg_map** out) {
  return guard([&] {
    check_ptr(ctx, "ctx");
    check_ptr(out, "out");
    require(window > 0, TLG_INVALID_ARGUMENT, "window must be positive");
    *out = map_new(ctx, voxel_size, window);
  });
}

tlg_status tlg_map_destroy(tlg_map* m) {
  return guard([&] { map_free(m); });
}

tlg_status tlg_map_insert(tlg_map* m, const double* px, const double* py, const double* pz,
                          const uint8_t* kind, const int32_t* label, size_t n, tlg_mem mem,
                          const double R[9], const double t[3]) {
  return guard([&] {
    check_ptr(m, "map");
    check_ptr(R, "R");
    check_ptr(t, "t");
    tlg_ctx* ctx = map_ctx(m);
    const double* dx = as_device(ctx, S_IN_HX, px, n, mem);
    const double* dy = as_device(ctx, S_IN_HY, py, n, mem);
    const double* dz = as_device(ctx, S_IN_HZ, pz, n, mem);
    const uint8_t* dk = as_device(ctx, S_MOMENT_ROW, kind, n, mem);
    const int32_t* dl = label ? as_device(ctx, S_IN_X, label, n, mem) : nullptr;
    map_insert(m, dx, dy, dz, dk, dl, n, R, t);
  });
}

tlg_status tlg_map_points(tlg_map* m, int kind, double* xyz, int32_t* labels, size_t cap,
                          size_t* count) {
  return guard([&] {
    check_ptr(m, "map");
    require(kind == 0 || kind == 1, TLG_INVALID_ARGUMENT, "kind must be 0 (edge) or 1 (planar)");
    const size_t c = map_points_host(m, kind, xyz, labels, cap);
    if (count) *count = c;
  });
}

tlg_status tlg_build_correspondences(tlg_map* m, const double* px, const double* py,
                                     const double* pz, const uint8_t* kind, size_t n,
                                     tlg_mem mem, const double R[9], const double t[3],
                                     const tlg_match_config* cfg, size_t* count) {
  return guard([&] {
    check_ptr(m, "map");
    check_ptr(R, "R");
    check_ptr(t, "t");
    check_ptr(cfg, "cfg");
    require(cfg->corr_gate > 0.0, TLG_INVALID_ARGUMENT, "corr_gate must be positive");
    tlg_ctx* ctx = map_ctx(m);
    const double* dx = as_device(ctx, S_IN_HX, px, n, mem);
    const double* dy = as_device(ctx, S_IN_HY, py, n, mem);
    const double* dz = as_device(ctx, S_IN_HZ, pz, n, mem);
    const uint8_t* dk = as_device(ctx, S_MOMENT_ROW, kind, n, mem);
    const double v[11] = {cfg->corr_gate,      cfg->huber_delta,   cfg->plane_fit_tol,
                          cfg->plane_eig_ratio, cfg->edge_eig_ratio, cfg->edge_fit_tol,
                          cfg->edge_min_extent, cfg->trim_ratio,    cfg->trim_floor,
                          cfg->ground_corr_voxel, cfg->ground_corr_radius};
    const size_t c = build_correspondences_device(m, dx, dy, dz, dk, n, R, t, v);
    if (count) *count = c;
  });
}

tlg_status tlg_correspondences_get(tlg_map* m, int32_t* kind, uint32_t* feature, double* params,
                                   double* weight, int32_t* label, double* dist, double* fitq,
                                   size_t cap) {
  return guard([&] {
    check_ptr(m, "map");
    correspondences_host(m, kind, feature, params, weight, label, dist, fitq, cap);
  });
}

tlg_status tlg_feature_rows(tlg_ctx* ctx, const int32_t* kind, const double* p_sensor,
                            const double* params, const double* weight, size_t n,
                            const double R[9], const double t[3], double* r, double* J,
                            size_t cap_rows, size_t* rows) {
  return guard([&] {
    check_ptr(ctx, "ctx");
    check_ptr(R, "R");
    check_ptr(t, "t");
    check_ptr(rows, "rows");
    size_t need = 0;
    for (size_t j = 0; j < n; ++j) need += kind[j] == 0 ? 3 : 1;
    *rows = need;
    if (need > cap_rows) throw Error(TLG_BUFFER_TOO_SMALL, "feature rows: buffer too small");
    size_t got = 0;
    feature_rows_device(ctx, n, kind, p_sensor, params, weight, R, t, r, J, &got);
  });
}

tlg_status tlg_feature_normal_eq(tlg_map* m, const double R[9], const double t[3],
                                 tlg_normal_eq* ne) {
  return guard([&] {
    check_ptr(m, "map");
    check_ptr(R, "R");
    check_ptr(t, "t");
    check_ptr(ne, "ne");
    double h[29];
    feature_normal_eq_device(m, R, t, h);
    for (int k = 0; k < 21; ++k) ne->A[k] = h[k];
    for (int k = 0; k < 6; ++k) ne->g[k] = h[21 + k];
    ne->cost = h[27];
    ne->valid = h[28];
  });
}


tlg_status tlg_kernel_finalize(tlg_kernel_params* p) {
  return guard([&] {
    check_ptr(p, "params");
    finalize_kernel(*p);
  });
}

// kernel.cpp:27-35, elementwise: (x - c).squaredNorm() without contraction,
// the `>` cutoff test, exp(-r2 / (2 b b)); non-finite inputs raise a flag.
__global__ void k_kernel_eval(const double* __restrict__ x, const double* __restrict__ y,
                              const double* __restrict__ cx, const double* __restrict__ cy,
                              size_t n, double cut2, double denom, double* __restrict__ out,
                              int* __restrict__ bad) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const double xi = x[i], yi = y[i], ci = cx[i], di = cy[i];
    if (!isfinite(xi) || !isfinite(yi) || !isfinite(ci) || !isfinite(di)) {
      atomicOr(bad, 1);
      out[i] = 0.0;
      continue;
    }
    const double dx = __dsub_rn(xi, ci), dy = __dsub_rn(yi, di);
    const double r2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
    out[i] = (r2 > cut2) ? 0.0 : exp(__ddiv_rn(-r2, denom));
  }
}

tlg_status tlg_kernel_eval(tlg_ctx* ctx, const tlg_kernel_params* p, const double* x,
                           const double* y, const double* cx, const double* cy, size_t n,
                           tlg_mem in_mem, double bandwidth, double* out, tlg_mem out_mem) {
  return guard([&] {
    check_ptr(ctx, "ctx");
    check_ptr(p, "params");
    if (!std::isfinite(bandwidth)) throw Error(TLG_DOMAIN_ERROR, "non-finite kernel input");
    if (!(bandwidth > 0.0)) throw Error(TLG_DOMAIN_ERROR, "bandwidth must be > 0");
    if (n == 0) return;
    check_ptr(x, "x");
    check_ptr(y, "y");
    check_ptr(cx, "cx");
    check_ptr(cy, "cy");
    check_ptr(out, "out");
    const double* dx = as_device(ctx, S_IN_X, x, n, in_mem);
    const double* dy = as_device(ctx, S_IN_Y, y, n, in_mem);
    const double* dcx = as_device(ctx, S_IN_HX, cx, n, in_mem);
    const double* dcy = as_device(ctx, S_IN_HY, cy, n, in_mem);
    const bool dev = out_mem == TLG_DEVICE;
    double* dout = dev ? out : ctx->ws<double>(S_OUT_Z, n);
    int* bad = ctx->ws<int>(S_FLAGS, 1);
    TLG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
    const double denom = 2.0 * bandwidth * bandwidth;
    const int grid = static_cast<int>(std::min<size_t>((n + 255) / 256, size_t(ctx->num_sms) * 8));
    k_kernel_eval<<<grid, 256, 0, ctx->stream>>>(dx, dy, dcx, dcy, n, p->cutoff_radius * p->cutoff_radius,
                                                denom, dout, bad);
    TLG_LAUNCHED(ctx);
    int hbad = 0;
    TLG_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    if (hbad) throw Error(TLG_DOMAIN_ERROR, "non-finite kernel input");
    if (!dev) {
      copy_out(ctx, out, dout, n * 8, TLG_HOST);
      ctx->sync();
    }
  });
}

// ---- center selection ------------------------------------------------------
static tlg_status select_impl(tlg_ctx* ctx, const double* x, const double* y, const double* z,
                              size_t m, size_t zn, tlg_mem in_mem, const tlg_center_params* p,
                              double* out_x, double* out_y, size_t cap, size_t* out_n,
                              tlg_mem out_mem, bool throw_empty) {
  return guard([&] {
    check_ptr(ctx, "ctx");
    check_ptr(p, "params");
    check_ptr(out_n, "out_n");
    *out_n = 0;
    // center_select.cpp:22-24 then :25 (validate)
    if (!(p->mesh_resolution > 0.0))
      throw Error(TLG_INVALID_ARGUMENT, "mesh_resolution must be > 0");
    if (p->accept_count < 1) throw Error(TLG_INVALID_ARGUMENT, "accept_count must be >= 1");
    const double* dx = as_device(ctx, S_IN_X, x, m, in_mem);
    const double* dy = as_device(ctx, S_IN_Y, y, m, in_mem);
    const double* dz = as_device(ctx, S_IN_Z, z, zn, in_mem);
    validate_obs_device(ctx, dx, dy, dz, m, zn);
    const double *nx = nullptr, *ny = nullptr;
    const size_t n = supported_nodes_device(ctx, dx, dy, m, *p, &nx, &ny);
    *out_n = n;
    if (throw_empty && n == 0) throw NoSupported();
    if (n > cap) throw Error(TLG_BUFFER_TOO_SMALL, "output buffer too small");
    if (n) {
      check_ptr(out_x, "out_x");
      check_ptr(out_y, "out_y");
      copy_out(ctx, out_x, nx, n * 8, out_mem);
      copy_out(ctx, out_y, ny, n * 8, out_mem);
    }
    ctx->sync();
  });
}

tlg_status tlg_supported_mesh_nodes(tlg_ctx* ctx, const double* x, const double* y,
                                    const double* z, size_t m, size_t z_len, tlg_mem in_mem,
                                    const tlg_center_params* params, double* out_x,
                                    double* out_y, size_t cap, size_t* out_n, tlg_mem out_mem) {
  return select_impl(ctx, x, y, z, m, z_len, in_mem, params, out_x, out_y, cap, out_n, out_mem,
                     false);
}

tlg_status tlg_select_centers(tlg_ctx* ctx, const double* x, const double* y, const double* z,
                              size_t m, size_t z_len, tlg_mem in_mem,
                              const tlg_center_params* params, double* out_x, double* out_y,
                              size_t cap, size_t* out_n, tlg_mem out_mem) {
  return select_impl(ctx, x, y, z, m, z_len, in_mem, params, out_x, out_y, cap, out_n, out_mem,
                     true);
}

// ---- model -------------------------------------------------------------------
tlg_status tlg_model_create(tlg_ctx* ctx, const tlg_kernel_params* kernel,
                            const tlg_center_params* centers, const double* cx,
                            const double* cy, size_t n, tlg_mem mem, tlg_model** out) {
  return guard([&] {
    check_ptr(ctx, "ctx");
    check_ptr(kernel, "kernel");
    check_ptr(centers, "centers");
    check_ptr(out, "out");
    std::vector<double> hx(n), hy(n);
    if (n) {
      check_ptr(cx, "cx");
      check_ptr(cy, "cy");
      if (mem == TLG_DEVICE) {
        TLG_CUDA(cudaMemcpy(hx.data(), cx, n * 8, cudaMemcpyDeviceToHost));
        TLG_CUDA(cudaMemcpy(hy.data(), cy, n * 8, cudaMemcpyDeviceToHost));
      } else {
        std::memcpy(hx.data(), cx, n * 8);
        std::memcpy(hy.data(), cy, n * 8);
      }
    }
    *out = model_create_impl(ctx, *kernel, *centers, hx.data(), hy.data(), n);
  });
}

tlg_status tlg_model_destroy(tlg_model* m) {
  return guard([&] {
    if (!m) return;
    cudaStreamSynchronize(m->ctx->stream);
    delete m;
  });
}

tlg_status tlg_model_counts(const tlg_model* m, size_t* nc, size_t* nb) {
  return guard([&] {
    check_ptr(m, "model");
    if (nc) *nc = m->hcx.size();
    if (nb) *nb = m->members.size();
  });
}

tlg_status tlg_model_sweep(tlg_model* m, int* kind, int* exp_recurrence) {
  return guard([&] {
    check_ptr(m, "model");
    ensure_grid(m);
    if (kind) *kind = sweep_kind(m);
    if (exp_recurrence) *exp_recurrence = m->lat.valid ? lattice_view(m).rec_ok : 0;
  });
}

tlg_status tlg_model_set_exact_cutoff(tlg_model* m, int exact) {
  return guard([&] {
    check_ptr(m, "model");
    m->exact_cutoff = exact != 0;
  });
}

tlg_status tlg_model_kernel(const tlg_model* m, tlg_kernel_params* out) {
  return guard([&] {
    check_ptr(m, "model");
    check_ptr(out, "out");
    *out = m->kernel;
  });
}

tlg_status tlg_model_center_params(const tlg_model* m, tlg_center_params* out) {
  return guard([&] {
    check_ptr(m, "model");
    check_ptr(out, "out");
    *out = m->cparams;
  });
}

tlg_status tlg_model_get_centers(tlg_model* m, double* cx, double* cy, tlg_mem mem) {
  return guard([&] {
    check_ptr(m, "model");
    const size_t n = m->hcx.size();
    if (cx) copy_out(m->ctx, cx, m->cx.p, n * 8, mem);
    if (cy) copy_out(m->ctx, cy, m->cy.p, n * 8, mem);
    m->ctx->sync();
  });
}

tlg_status tlg_model_get_weights(tlg_model* m, double* w, tlg_mem mem) {
  return guard([&] {
    check_ptr(m, "model");
    check_ptr(w, "w");
    copy_out(m->ctx, w, m->w.p, m->hcx.size() * 8, mem);
    m->ctx->sync();
  });
}

tlg_status tlg_model_set_weights(tlg_model* m, const double* w, tlg_mem mem) {
  return guard([&] {
    check_ptr(m, "model");
    check_ptr(w, "w");
    copy_in(m->ctx, m->w.p, w, m->hcx.size() * 8, mem);
    sync_weights_to_grid(m);
    m->ctx->sync();
  });
}

tlg_status tlg_model_get_block_index(tlg_model* m, uint32_t* out, tlg_mem mem) {
  return guard([&] {
    check_ptr(m, "model");
    check_ptr(out, "out");
    copy_out(m->ctx, out, m->d_block_index.p, m->hcx.size() * 4, mem);
    m->ctx->sync();
  });
}

tlg_status tlg_model_block_size(const tlg_model* m, uint32_t b, size_t* n) {
  return guard([&] {
    check_ptr(m, "model");
    check_ptr(n, "n");
    require(b < m->members.size(), TLG_INVALID_ARGUMENT, "block id out of range");
    *n = m->members[b].size();
  });
}

tlg_status tlg_model_get_block_members(const tlg_model* m, uint32_t b, uint32_t* out) {
  return guard([&] {
    check_ptr(m, "model");
    require(b < m->members.size(), TLG_INVALID_ARGUMENT, "block id out of range");
    if (!m->members[b].empty()) {
      check_ptr(out, "out");
      std::memcpy(out, m->members[b].data(), m->members[b].size() * 4);
    }
  });
}

tlg_status tlg_model_get_block_info_inverse(tlg_model* m, uint32_t b, double* out, tlg_mem mem) {
  return guard([&] {
    check_ptr(m, "model");
    require(b < m->members.size(), TLG_INVALID_ARGUMENT, "block id out of range");
    const size_t bn = m->members[b].size();
    if (!bn) return;
    check_ptr(out, "out");
    TLG_CUDA(cudaMemcpy2DAsync(out, bn * 8, m->pool.p + m->blk_off[b], m->blk_ld[b] * 8, bn * 8,
                               bn, mem == TLG_DEVICE ? cudaMemcpyDeviceToDevice
                                                     : cudaMemcpyDeviceToHost,
                               m->ctx->stream));
    m->ctx->sync();
  });
}

tlg_status tlg_model_set_block_info_inverse(tlg_model* m, uint32_t b, const double* in,
                                            tlg_mem mem) {
  return guard([&] {
    check_ptr(m, "model");
    require(b < m->members.size(), TLG_INVALID_ARGUMENT, "block id out of range");
    const size_t bn = m->members[b].size();
    if (!bn) return;
    check_ptr(in, "in");
    TLG_CUDA(cudaMemcpy2DAsync(m->pool.p + m->blk_off[b], m->blk_ld[b] * 8, in, bn * 8, bn * 8,
                               bn, mem == TLG_DEVICE ? cudaMemcpyDeviceToDevice
                                                     : cudaMemcpyHostToDevice,
                               m->ctx->stream));
    m->ctx->sync();
  });
}

tlg_status tlg_eval(tlg_model* m, const double* x, const double* y, size_t n, tlg_mem in_mem,
                    double* z, uint8_t* supported, double* gx, double* gy, tlg_mem out_mem) {
  return guard([&] {
    check_ptr(m, "model");
    if (n == 0) return;
    check_ptr(x, "x");
    check_ptr(y, "y");
    tlg_ctx* ctx = m->ctx;
    const double* dx = as_device(ctx, S_IN_X, x, n, in_mem);
    const double* dy = as_device(ctx, S_IN_Y, y, n, in_mem);
    const bool dev = out_mem == TLG_DEVICE;
    double* dz = z ? (dev ? z : ctx->ws<double>(S_OUT_Z, n)) : nullptr;
    uint8_t* ds = supported ? (dev ? supported : ctx->ws<uint8_t>(S_OUT_SUP, n)) : nullptr;
    double* dgx = gx ? (dev ? gx : ctx->ws<double>(S_OUT_GX, n)) : nullptr;
    double* dgy = gy ? (dev ? gy : ctx->ws<double>(S_OUT_GY, n)) : nullptr;
    eval_device(m, dx, dy, n, dz, ds, dgx, dgy);
    if (!dev) {
      if (z) copy_out(ctx, z, dz, n * 8, TLG_HOST);
      if (supported) copy_out(ctx, supported, ds, n, TLG_HOST);
      if (gx) copy_out(ctx, gx, dgx, n * 8, TLG_HOST);
      if (gy) copy_out(ctx, gy, dgy, n * 8, TLG_HOST);
      ctx->sync();
    }
  });
}

tlg_status tlg_moment_features(tlg_model* m, const double* x, const double* y, size_t n,
                               tlg_mem in_mem, uint32_t* row_ptr, uint32_t* ids, double* vals,
                               size_t cap, size_t* nnz, tlg_mem out_mem) {
  return guard([&] {
    check_ptr(m, "model");
    check_ptr(nnz, "nnz");
    *nnz = 0;
    if (n == 0) return;
    tlg_ctx* ctx = m->ctx;
    const double* dx = as_device(ctx, S_IN_X, x, n, in_mem);
    const double* dy = as_device(ctx, S_IN_Y, y, n, in_mem);
    uint32_t* drow = ctx->ws<uint32_t>(S_MOMENT_ROW, n + 1);
    uint32_t* dids = nullptr;
    double* dvals = nullptr;
    moment_device(m, dx, dy, n, drow, &dids, &dvals, nnz);
    if (*nnz > cap) throw Error(TLG_BUFFER_TOO_SMALL, "output buffer too small");
    if (row_ptr) copy_out(ctx, row_ptr, drow, (n + 1) * 4, out_mem);
    if (ids) copy_out(ctx, ids, dids, *nnz * 4, out_mem);
    if (vals) copy_out(ctx, vals, dvals, *nnz * 8, out_mem);
    ctx->sync();
  });
}

tlg_status tlg_manifold_rows(tlg_model* m, const double R[9], const double t[3], const double* hx,
                             const double* hy, const double* hz, size_t n, tlg_mem in_mem,
                             double wheel_radius, double lambda_M, double huber_delta, double* r,
                             double* J, uint8_t* valid, double* raw, tlg_mem out_mem,
                             tlg_normal_eq* ne) {
  return guard([&] {
    check_ptr(m, "model");
    check_ptr(R, "R");
    check_ptr(t, "t");
    require(lambda_M >= 0.0, TLG_INVALID_ARGUMENT, "lambda_M must be >= 0");
    if (n == 0) {
      if (ne) *ne = tlg_normal_eq{};
      return;
    }
    tlg_ctx* ctx = m->ctx;
    const bool dev = out_mem == TLG_DEVICE;
    if (in_mem == TLG_HOST && n >= (size_t{1} << 20) && (dev || (!r && !J && !valid && !raw))) {
      // large host batches: H2D slices overlap the kernel on earlier slices
      manifold_device_streamed(m, R, t, hx, hy, hz, n, wheel_radius, lambda_M, huber_delta, r, J,
                               valid, raw, ne);
      return;
    }
    const double* dhx = as_device(ctx, S_IN_HX, hx, n, in_mem);
    const double* dhy = as_device(ctx, S_IN_HY, hy, n, in_mem);
    const double* dhz = as_device(ctx, S_IN_HZ, hz, n, in_mem);
    double* dr = r ? (dev ? r : ctx->ws<double>(S_OUT_R, n)) : nullptr;
    double* dJ = J ? (dev ? J : ctx->ws<double>(S_OUT_J, 6 * n)) : nullptr;
    uint8_t* dv = valid ? (dev ? valid : ctx->ws<uint8_t>(S_OUT_SUP, n)) : nullptr;
    double* draw = raw ? (dev ? raw : ctx->ws<double>(S_OUT_RAW, n)) : nullptr;
    manifold_device(m, R, t, dhx, dhy, dhz, n, wheel_radius, lambda_M, huber_delta, dr, dJ, dv,
                    draw, ne);
    if (!dev) {
      if (r) copy_out(ctx, r, dr, n * 8, TLG_HOST);
      if (J) copy_out(ctx, J, dJ, 6 * n * 8, TLG_HOST);
      if (valid) copy_out(ctx, valid, dv, n, TLG_HOST);
      if (raw) copy_out(ctx, raw, draw, n * 8, TLG_HOST);
      ctx->sync();
    }
  });
}

tlg_status tlg_scan_create(tlg_model* m, const double R0[9], const double t0[3], const double* hx,
                           const double* hy, const double* hz, size_t n, tlg_mem in_mem,
                           tlg_scan** out) {
  return guard([&] {
    check_ptr(m, "model");
    check_ptr(R0, "R0");
    check_ptr(t0, "t0");
    check_ptr(out, "out");
    tlg_ctx* ctx = m->ctx;
    const double* dhx = as_device(ctx, S_IN_HX, hx, n, in_mem);
    const double* dhy = as_device(ctx, S_IN_HY, hy, n, in_mem);
    const double* dhz = as_device(ctx, S_IN_HZ, hz, n, in_mem);
    *out = scan_create(m, R0, t0, dhx, dhy, dhz, n);
  });
}

tlg_status tlg_scan_destroy(tlg_scan* scan) {
  return guard([&] {
    if (!scan) return;
    cudaStreamSynchronize(scan->ctx->stream);
    delete scan;
  });
}

tlg_status tlg_scan_info(const tlg_scan* scan, size_t* n, double* bin_ms) {
  return guard([&] {
    check_ptr(scan, "scan");
    if (n) *n = scan->n;
    if (bin_ms) *bin_ms = scan->bin_ms;
  });
}

tlg_status tlg_scan_permutation(tlg_scan* scan, uint32_t* perm, tlg_mem out_mem) {
  return guard([&] {
    check_ptr(scan, "scan");
    check_ptr(perm, "perm");
    copy_out(scan->ctx, perm, scan->perm.p, scan->n * 4, out_mem);
    scan->ctx->sync();
  });
}

tlg_status tlg_scan_manifold_rows(tlg_model* m, tlg_scan* scan, const double R[9],
                                  const double t[3], double wheel_radius, double lambda_M,
                                  double huber_delta, double* r, double* J, uint8_t* valid,
                                  double* raw, tlg_mem out_mem, tlg_normal_eq* ne) {
  return tlg_manifold_rows(m, R, t, scan ? scan->hx.p : nullptr, scan ? scan->hy.p : nullptr,
                           scan ? scan->hz.p : nullptr, scan ? scan->n : 0, TLG_DEVICE,
                           wheel_radius, lambda_M, huber_delta, r, J, valid, raw, out_mem, ne);
}

tlg_status tlg_recursive_update(tlg_model* m, const double* x, const double* y, const double* z,
                                size_t mm, size_t z_len, tlg_mem in_mem, int allow_birth,
                                tlg_update_report* report) {
  return guard([&] {
    check_ptr(m, "model");
    tlg_ctx* ctx = m->ctx;
    tlg_update_report rep{};
    const double* dx = as_device(ctx, S_IN_X, x, mm, in_mem);
    const double* dy = as_device(ctx, S_IN_Y, y, mm, in_mem);
    const double* dz = as_device(ctx, S_IN_Z, z, z_len, in_mem);
    const int* vflag = validate_obs_launch(ctx, dx, dy, dz, mm, z_len);
    recursive_update_device(m, dx, dy, dz, mm, allow_birth != 0, &rep, vflag);
    if (report) *report = rep;
  });
}

tlg_status tlg_fit_batch_ridge(tlg_ctx* ctx, const tlg_kernel_params* kernel,
                               const tlg_center_params* centers, const double* cx,
                               const double* cy, size_t n, const double* x, const double* y,
                               const double* z, size_t m, size_t z_len, tlg_mem mem,
                               tlg_model** out) {
  tlg_model* model = nullptr;
  tlg_status st = guard([&] {
    check_ptr(out, "out");
    // terrain_model.cpp:272 validates before building the model
    const double* dx = as_device(ctx, S_IN_X, x, m, mem);
    const double* dy = as_device(ctx, S_IN_Y, y, m, mem);
    const double* dz = as_device(ctx, S_IN_Z, z, z_len, mem);
    validate_obs_device(ctx, dx, dy, dz, m, z_len);
  });
  if (st != TLG_OK) return st;
  st = tlg_model_create(ctx, kernel, centers, cx, cy, n, mem, &model);
  if (st != TLG_OK) return st;
  st = guard([&] {
    const double* dx = as_device(ctx, S_IN_X, x, m, mem);
    const double* dy = as_device(ctx, S_IN_Y, y, m, mem);
    const double* dz = as_device(ctx, S_IN_Z, z, z_len, mem);
    batch_fit_device(model, dx, dy, dz, m);
  });
  if (st != TLG_OK) {
    tlg_model_destroy(model);
    return st;
  }
  *out = model;
  return TLG_OK;
}

// ---- point-sharded batch ridge -------------------------------------
tlg_status tlg_batch_ridge_system(tlg_model* m, size_t* n, size_t* ld, size_t* elems) {
  return guard([&] {
    check_ptr(m, "model");
    check_ptr(n, "n");
    check_ptr(ld, "ld");
    check_ptr(elems, "elems");
    ensure_grid(m);
    batch_system_dims(m, n, ld, elems);
  });
}

tlg_status tlg_batch_ridge_assemble(tlg_model* m, const double* x, const double* y,
                                    const double* z, size_t mm, tlg_mem mem, double* H, size_t ld,
                                    double* b, int add_lambda) {
  return guard([&] {
    check_ptr(m, "model");
    check_ptr(H, "H");
    check_ptr(b, "b");
    tlg_ctx* ctx = m->ctx;
    const double* dx = nullptr;
    const double* dy = nullptr;
    const double* dz = nullptr;
    if (mm) {  // a shard may be empty
      dx = as_device(ctx, S_IN_X, x, mm, mem);
      dy = as_device(ctx, S_IN_Y, y, mm, mem);
      dz = as_device(ctx, S_IN_Z, z, mm, mem);
      validate_obs_device(ctx, dx, dy, dz, mm, mm);
    }
    batch_assemble_device(m, dx, dy, dz, mm, H, ld, b, add_lambda != 0);
  });
}

tlg_status tlg_batch_ridge_pattern(tlg_model* m, size_t* nnz) {
  return guard([&] {
    check_ptr(m, "model");
    check_ptr(nnz, "nnz");
    *nnz = batch_pattern_device(m);
  });
}

tlg_status tlg_batch_ridge_pack(tlg_model* m, const double* H, double* packed) {
  return guard([&] {
    check_ptr(m, "model");
    check_ptr(H, "H");
    check_ptr(packed, "packed");
    batch_pack_device(m, H, packed);
  });
}

tlg_status tlg_batch_ridge_unpack(tlg_model* m, const double* packed, double* H) {
  return guard([&] {
    check_ptr(m, "model");
    check_ptr(H, "H");
    check_ptr(packed, "packed");
    batch_unpack_device(m, packed, H);
  });
}

tlg_status tlg_batch_ridge_solve(tlg_model* m, double* H, size_t ld, double* b) {
  return guard([&] {
    check_ptr(m, "model");
    check_ptr(H, "H");
    check_ptr(b, "b");
    batch_solve_device(m, H, ld, b);
  });
}

// ---- RBFT snapshot (snapshot.cpp:7-126) ---------------------------------------
tlg_status tlg_model_save(tlg_model* m, const char* path) {
  return guard([&] {
    check_ptr(m, "model");
    check_ptr(path, "path");
    const size_t n = m->hcx.size();
    std::vector<double> w(n);
    if (n) {
      TLG_CUDA(cudaMemcpyAsync(w.data(), m->w.p, n * 8, cudaMemcpyDeviceToHost, m->ctx->stream));
    }
    std::vector<std::vector<double>> blocks(m->members.size());
    for (size_t b = 0; b < m->members.size(); ++b) {
      const size_t bn = m->members[b].size();
      blocks[b].resize(bn * bn);
      if (bn)
        TLG_CUDA(cudaMemcpy2DAsync(blocks[b].data(), bn * 8, m->pool.p + m->blk_off[b],
                                   m->blk_ld[b] * 8, bn * 8, bn, cudaMemcpyDeviceToHost,
                                   m->ctx->stream));
    }
    m->ctx->sync();
    std::ofstream out(path, std::ios::binary);
    if (!out) throw Error(TLG_RUNTIME_ERROR, std::string("cannot open ") + path);
    auto put32 = [&](uint32_t v) { out.write(reinterpret_cast<const char*>(&v), 4); };
    auto putd = [&](double v) { out.write(reinterpret_cast<const char*>(&v), 8); };
    out.write("RBFT", 4);
    put32(1u);
    put32(static_cast<uint32_t>(n));
    put32(static_cast<uint32_t>(m->members.size()));
    for (size_t i = 0; i < n; ++i) {
      putd(m->hcx[i]);
      putd(m->hcy[i]);
    }
    for (size_t i = 0; i < n; ++i) putd(w[i]);
    for (size_t i = 0; i < n; ++i) put32(m->block_index[i]);
    for (size_t b = 0; b < m->members.size(); ++b) {
      const size_t bn = m->members[b].size();
      for (size_t r = 0; r < bn; ++r)
        for (size_t c = 0; c <= r; ++c) putd(blocks[b][c * bn + r]);  // row-major lower
    }
    putd(m->kernel.sigma);
    putd(m->kernel.sigma_eps);
    putd(m->kernel.lambda);
    putd(m->kernel.cutoff_radius);
    putd(m->cparams.mesh_resolution);
    putd(m->cparams.accept_radius);
    put32(static_cast<uint32_t>(m->cparams.accept_count));
    putd(m->cparams.roi_min_x);
    putd(m->cparams.roi_min_y);
    putd(m->cparams.roi_max_x);
    putd(m->cparams.roi_max_y);
    if (!out) throw Error(TLG_RUNTIME_ERROR, std::string("write failed: ") + path);
  });
}

tlg_status tlg_model_load(tlg_ctx* ctx, const char* path, tlg_model** out) {
  tlg_model* model = nullptr;
  tlg_status st = guard([&] {
    check_ptr(ctx, "ctx");
    check_ptr(path, "path");
    check_ptr(out, "out");
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    if (!in) throw Error(TLG_RUNTIME_ERROR, std::string("cannot open ") + path);
    // one read of the whole file, then parse from memory
    const std::streamsize fsize = in.tellg();
    std::vector<char> buf(static_cast<size_t>(std::max<std::streamsize>(fsize, 0)));
    in.seekg(0);
    if (fsize > 0 && !in.read(buf.data(), fsize))
      throw Error(TLG_RUNTIME_ERROR, std::string("cannot read ") + path);
    size_t pos = 0;
    auto take = [&](void* dst, size_t nbytes) {
      if (pos + nbytes > buf.size()) throw Error(TLG_RUNTIME_ERROR, "truncated terrain snapshot");
      std::memcpy(dst, buf.data() + pos, nbytes);
      pos += nbytes;
    };
    auto get32 = [&]() {
      uint32_t v;
      take(&v, 4);
      return v;
    };
    auto getd = [&]() {
      double v;
      take(&v, 8);
      return v;
    };
    if (buf.size() < 4 || std::memcmp(buf.data(), "RBFT", 4) != 0)
      throw Error(TLG_RUNTIME_ERROR, std::string("not a terrain snapshot: ") + path);
    pos = 4;
    if (get32() != 1u) throw Error(TLG_RUNTIME_ERROR, "unsupported snapshot version");
    const uint32_t n = get32(), nb = get32();
    std::vector<double> cx(n), cy(n), w(n);
    for (uint32_t i = 0; i < n; ++i) {
      cx[i] = getd();
      cy[i] = getd();
    }
    for (uint32_t i = 0; i < n; ++i) w[i] = getd();
    std::vector<uint32_t> bidx(n);
    std::vector<std::vector<uint32_t>> mem(nb);
    for (uint32_t i = 0; i < n; ++i) {
      bidx[i] = get32();
      if (bidx[i] >= nb) throw Error(TLG_RUNTIME_ERROR, "corrupt block index");
      mem[bidx[i]].push_back(i);
    }
    std::vector<std::vector<double>> blocks(nb);
    for (uint32_t b = 0; b < nb; ++b) {
      const size_t bn = mem[b].size();
      blocks[b].resize(bn * bn);
      for (size_t r = 0; r < bn; ++r)
        for (size_t c = 0; c <= r; ++c) {
          const double v = getd();
          blocks[b][c * bn + r] = v;
          blocks[b][r * bn + c] = v;
        }
    }
    tlg_kernel_params k;
    k.sigma = getd();
    k.sigma_eps = getd();
    k.lambda = getd();
    k.cutoff_radius = getd();
    tlg_center_params cp{};
    cp.mesh_resolution = getd();
    cp.accept_radius = getd();
    cp.accept_count = static_cast<int32_t>(get32());
    cp.roi_min_x = getd();
    cp.roi_min_y = getd();
    cp.roi_max_x = getd();
    cp.roi_max_y = getd();
    // Build with the stored block structure: the snapshot's block ids are
    // authoritative (snapshot.cpp:89-96,120-123).
    model = model_create_impl(ctx, k, cp, nullptr, nullptr, 0);
    model->members = mem;
    model->block_index = bidx;
    model->blk_off.assign(nb, 0);
    model->blk_ld.assign(nb, 0);
    model->tile_blocks.clear();
    for (uint32_t i = 0; i < n; ++i) model->tile_blocks.emplace(tile_key(model, cx[i], cy[i]), bidx[i]);
    model->hcx = cx;
    model->hcy = cy;
    for (uint32_t i = 0; i < n; ++i) model->occupancy.insert(mesh_node_key(model, cx[i], cy[i]));
    size_t total = 0;
    for (uint32_t b = 0; b < nb; ++b) {
      const int ld = std::max(8, (static_cast<int>(mem[b].size()) + 7) & ~7);
      model->blk_ld[b] = ld;
      model->blk_off[b] = total;
      total += static_cast<size_t>(ld) * ld;
    }
    model->pool.ensure(total + total / 2 + 64);
    model->pool_used = total;
    upload_new_centres(model, 0);
    TLG_CUDA(cudaMemcpyAsync(model->w.p, w.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
    for (uint32_t b = 0; b < nb; ++b) {
      const size_t bn = mem[b].size();
      if (bn)
        TLG_CUDA(cudaMemcpy2DAsync(model->pool.p + model->blk_off[b], model->blk_ld[b] * 8,
                                   blocks[b].data(), bn * 8, bn * 8, bn, cudaMemcpyHostToDevice,
                                   ctx->stream));
    }
    ctx->sync();
    build_center_grid(model);
    ctx->sync();
  });
  if (st != TLG_OK) {
    delete model;
    return st;
  }
  *out = model;
  return TLG_OK;
}

}  // extern "C"

// ---- Communicator (SURVEY §8b tlg_comm_init) -------------------------------
// NCCL is resolved at tlg_comm_init with dlopen("libnccl.so.2"), preferring a
// copy the process already loaded (torch's), so the library itself never
// links NCCL and single-GPU users never need it.
namespace {
struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl_api() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.init_rank = reinterpret_cast<decltype(a.init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.destroy = reinterpret_cast<decltype(a.destroy)>(dlsym(h, "ncclCommDestroy"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    return a;
  }();
  require(api.get_unique_id && api.init_rank && api.all_reduce && api.destroy,
          TLG_RUNTIME_ERROR, "NCCL (libnccl.so.2) is not available");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* e = nccl_api().error_string ? nccl_api().error_string(r) : "?";
    throw Error(TLG_RUNTIME_ERROR, std::string(what) + ": " + e);
  }
}
}  // namespace

struct tlg_comm {
  tlg_ctx* ctx = nullptr;
  ncclComm_t comm = nullptr;
  int rank = 0, size = 1;
};

extern "C" {

tlg_status tlg_comm_unique_id(void* id) {
  return guard([&] {
    check_ptr(id, "id");
    static_assert(sizeof(ncclUniqueId) == TLG_COMM_ID_BYTES, "NCCL unique id size");
    ncclUniqueId u;
    nccl_check(nccl_api().get_unique_id(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
  });
}

tlg_status tlg_comm_init(tlg_ctx* ctx, const void* id, int rank, int size, tlg_comm** out) {
  return guard([&] {
    check_ptr(ctx, "ctx");
    check_ptr(id, "id");
    check_ptr(out, "out");
    require(size >= 1 && rank >= 0 && rank < size, TLG_INVALID_ARGUMENT, "bad rank / size");
    TLG_CUDA(cudaSetDevice(ctx->device));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    auto* c = new tlg_comm();
    c->ctx = ctx;
    c->rank = rank;
    c->size = size;
    const ncclResult_t r = nccl_api().init_rank(&c->comm, size, u, rank);
    if (r != ncclSuccess) {
      delete c;
      nccl_check(r, "ncclCommInitRank");
    }
    *out = c;
  });
}

tlg_status tlg_comm_destroy(tlg_comm* c) {
  return guard([&] {
    if (!c) return;
    if (c->comm) nccl_api().destroy(c->comm);
    delete c;
  });
}

tlg_status tlg_comm_allreduce_normal_eq(tlg_comm* c, tlg_normal_eq* ne) {
  return guard([&] {
    check_ptr(c, "comm");
    check_ptr(ne, "ne");
    if (c->size == 1) return;
    tlg_ctx* ctx = c->ctx;
    static_assert(sizeof(tlg_normal_eq) == 29 * sizeof(double), "29-double block");
    double* d = ctx->ws<double>(S_PARTIALS, 29);
    double* h = static_cast<double*>(ctx->host_stage(29 * sizeof(double)));
    std::memcpy(h, ne, sizeof(*ne));
    TLG_CUDA(cudaMemcpyAsync(d, h, sizeof(*ne), cudaMemcpyHostToDevice, ctx->stream));
    nccl_check(nccl_api().all_reduce(d, d, 29, ncclFloat64, ncclSum, c->comm, ctx->stream),
               "ncclAllReduce");
    TLG_CUDA(cudaMemcpyAsync(h, d, sizeof(*ne), cudaMemcpyDeviceToHost, ctx->stream));
    TLG_CUDA(cudaStreamSynchronize(ctx->stream));
    std::memcpy(ne, h, sizeof(*ne));
  });
}

tlg_status tlg_fit_batch_ridge_sharded(tlg_model* m, tlg_comm* c, const double* x, const double* y,
                                       const double* z, size_t mm, tlg_mem mem) {
  return guard([&] {
    check_ptr(m, "model");
    check_ptr(c, "comm");
    require(c->ctx == m->ctx, TLG_INVALID_ARGUMENT, "model and communicator on different contexts");
    tlg_ctx* ctx = m->ctx;
    ensure_grid(m);
    size_t n = 0, ld = 0, elems = 0;
    batch_system_dims(m, &n, &ld, &elems);
    if (n == 0) return;
    const double* dx = nullptr;
    const double* dy = nullptr;
    const double* dz = nullptr;
    if (mm) {
      dx = as_device(ctx, S_IN_X, x, mm, mem);
      dy = as_device(ctx, S_IN_Y, y, mm, mem);
      dz = as_device(ctx, S_IN_Z, z, mm, mem);
      validate_obs_device(ctx, dx, dy, dz, mm, mm);
    }
    double* H = ctx->ws<double>(S_HMAT, elems);
    double* b = ctx->ws<double>(S_WORK3, n);
    batch_assemble_device(m, dx, dy, dz, mm, H, ld, b, c->rank == 0);
    if (c->size > 1) {
      // the structural nonzeros only (tlg_batch_ridge_pack), then the rhs
      const size_t nnz = batch_pattern_device(m);
      double* P = ctx->ws<double>(S_GEMVPART, nnz);
      batch_pack_device(m, H, P);
      nccl_check(nccl_api().all_reduce(P, P, nnz, ncclFloat64, ncclSum, c->comm, ctx->stream),
                 "ncclAllReduce");
      batch_unpack_device(m, P, H);
      nccl_check(nccl_api().all_reduce(b, b, n, ncclFloat64, ncclSum, c->comm, ctx->stream),
                 "ncclAllReduce");
    }
    batch_solve_device(m, H, ld, b);
  });
}

}  // extern "C"

