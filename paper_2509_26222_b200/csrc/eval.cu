// K3 eval_height_grad and K4 manifold_rows_reduce.
//
// K3: predict_height / predict_gradient (terrain_model.cpp:109-143) per
//     query point. Neighbour membership replicates GridIndex2::radius_query
//     (grid_index.hpp:32-48) bit-exactly: same cell coordinates
//     floor(v / cell), same (2*span+1)^2 cell window, same no-FMA
//     r^2 = dx*dx + dy*dy <= cutoff^2 test. Values are FP64 with FMA
//     accumulation (parity: 1e-9 relative).
// K4: the manifold soft-constraint rows (contact.cpp:7-39 +
//     scan_matcher.cpp:221-248), materialised as r / J (column-major rows x 6)
//     / valid, with the 6x6 normal equations J^T J, J^T r and the cost reduced
//     in the same pass: per-thread register accumulators, warp shuffles, one
//     partial per CTA, then a fixed-order final reduction (deterministic, no
//     FP64 atomics).
#include <cmath>

#include "internal.cuh"

namespace tlg {

struct EvalOut {
  double z, sx, sy;  // sum w k, sum w k (c - x), sum w k (c - y)
  bool sup;
};

// Sweeps the reference's candidate cells of query (x, y); cells of one x
// column are contiguous in cell order, so each column is one index range.
__device__ __forceinline__ EvalOut eval_point(const GridView& g, double x, double y, double r2,
                                              double neg_inv_2b2) {
  EvalOut o{0.0, 0.0, 0.0, false};
  const int qx = static_cast<int>(floor(x / g.cell));
  const int qy = static_cast<int>(floor(y / g.cell));
  const int y_lo = max(qy - g.span - g.gy0, 0);
  const int y_hi = min(qy + g.span - g.gy0, g.gny - 1);
  if (y_lo > y_hi) return o;
  const int x_lo = max(qx - g.span - g.gx0, 0);
  const int x_hi = min(qx + g.span - g.gx0, g.gnx - 1);
  for (int gx = x_lo; gx <= x_hi; ++gx) {
    const int b = __ldg(g.cell_start + gx * g.gny + y_lo);
    const int e = __ldg(g.cell_start + gx * g.gny + y_hi + 1);
    for (int k = b; k < e; ++k) {
      const double cx = __ldg(g.cx + k), cy = __ldg(g.cy + k);
      const double dx = cx - x, dy = cy - y;
      const double d2 = sq2_exact(dx, dy);
      if (d2 <= r2) {
        const double wk = __ldg(g.w + k) * exp(d2 * neg_inv_2b2);
        o.z += wk;
        o.sx = fma(wk, dx, o.sx);
        o.sy = fma(wk, dy, o.sy);
        o.sup = true;
      }
    }
  }
  return o;
}

__global__ void __launch_bounds__(256) k_eval(GridView g, const double* __restrict__ x,
                                              const double* __restrict__ y, size_t n, double r2,
                                              double neg_inv_2s2, double inv_s2,
                                              double* __restrict__ z, uint8_t* __restrict__ sup,
                                              double* __restrict__ gx, double* __restrict__ gy,
                                              int* __restrict__ err) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const double px = x[i], py = y[i];
    if (!isfinite(px) || !isfinite(py)) {
      atomicOr(err, 1);
      continue;
    }
    const EvalOut o = eval_point(g, px, py, r2, neg_inv_2s2);
    if (z) z[i] = o.sup ? o.z : 0.0;
    if (sup) sup[i] = o.sup ? 1 : 0;
    if (gx) gx[i] = o.sx * inv_s2;
    if (gy) gy[i] = o.sy * inv_s2;
  }
}

static unsigned grid_for(tlg_ctx* ctx, size_t n, int threads, int per_sm) {
  const size_t want = (n + threads - 1) / threads;
  const size_t cap = static_cast<size_t>(ctx->num_sms) * per_sm;
  return static_cast<unsigned>(std::max<size_t>(1, std::min(want, cap)));
}

static void check_err_flag(tlg_ctx* ctx, int* d_err, tlg_status st, const char* msg) {
  int h = 0;
  TLG_CUDA(cudaMemcpyAsync(&h, d_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  TLG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h) throw Error(st, msg);
}

void eval_device(tlg_model* m, const double* x, const double* y, size_t n, double* z,
                 uint8_t* sup, double* gx, double* gy) {
  tlg_ctx* ctx = m->ctx;
  ensure_grid(m);
  int* err = ctx->ws<int>(S_FLAGS, 4);
  TLG_CUDA(cudaMemsetAsync(err, 0, sizeof(int), ctx->stream));
  if (n) {
    prof_begin(ctx, 1);
    k_eval<<<grid_for(ctx, n, 256, 8), 256, 0, ctx->stream>>>(
        grid_view(m), x, y, n, m->kc.r2, m->kc.neg_inv_2s2, m->kc.inv_s2, z, sup, gx, gy, err);
    TLG_LAUNCHED(ctx);
    prof_mark_end(ctx);
  }
  check_err_flag(ctx, err, TLG_DOMAIN_ERROR, "non-finite query");
  prof_collect(ctx);
}

// ---------------------------------------------------------------------------
// K4
struct Pose {
  double R[9];
  double t[3];
};

constexpr int kNE = 29;  // 21 (A upper) + 6 (g) + cost + valid
constexpr int kManifoldThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kManifoldThreads) k_manifold(
    GridView g, Pose pose, const double* __restrict__ hx, const double* __restrict__ hy,
    const double* __restrict__ hz, size_t n, double r2, double neg_inv_2s2, double inv_s2,
    double wheel_radius, double sl, double huber, double* __restrict__ out_r,
    double* __restrict__ out_J, uint8_t* __restrict__ out_valid, double* __restrict__ out_raw,
    double* __restrict__ partials, int* __restrict__ err) {
  double acc[kNE];
#pragma unroll
  for (int k = 0; k < kNE; ++k) acc[k] = 0.0;
  const double* R = pose.R;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const double h0 = hx[i], h1 = hy[i], h2 = hz[i];
    // xi = R h + t (leg_model.cpp:31, contact.cpp:183)
    const double xi0 = fma(R[2], h2, fma(R[1], h1, R[0] * h0)) + pose.t[0];
    const double xi1 = fma(R[5], h2, fma(R[4], h1, R[3] * h0)) + pose.t[1];
    const double xi2 = fma(R[8], h2, fma(R[7], h1, R[6] * h0)) + pose.t[2];
    double r = 0.0, raw = 0.0, J[6] = {0, 0, 0, 0, 0, 0};
    bool valid = false;
    if (!isfinite(xi0) || !isfinite(xi1)) {
      atomicOr(err, 1);
    } else {
      const EvalOut o = eval_point(g, xi0, xi1, r2, neg_inv_2s2);
      if (o.sup) {
        valid = true;
        raw = xi2 - wheel_radius - o.z;
        const double gxv = o.sx * inv_s2, gyv = o.sy * inv_s2;
        // dr/dxi = [-gx, -gy, 1]; J_theta = h x (R^T dr); J_t = dr
        const double u0 = fma(R[6], 1.0, fma(R[3], -gyv, R[0] * -gxv));
        const double u1 = fma(R[7], 1.0, fma(R[4], -gyv, R[1] * -gxv));
        const double u2 = fma(R[8], 1.0, fma(R[5], -gyv, R[2] * -gxv));
        double w = 1.0;
        const double a = fabs(raw);
        if (huber > 0.0 && a > huber) w = sqrt(huber / a);
        const double s = sl * w;
        r = s * raw;
        J[0] = s * fma(h1, u2, -h2 * u1);
        J[1] = s * fma(h2, u0, -h0 * u2);
        J[2] = s * fma(h0, u1, -h1 * u0);
        J[3] = s * -gxv;
        J[4] = s * -gyv;
        J[5] = s;
      }
    }
    if (out_r) out_r[i] = r;
    if (out_raw) out_raw[i] = raw;
    if (out_valid) out_valid[i] = valid ? 1 : 0;
    if (out_J) {
#pragma unroll
      for (int c = 0; c < 6; ++c) out_J[c * n + i] = J[c];
    }
    int k = 0;
#pragma unroll
    for (int a = 0; a < 6; ++a)
#pragma unroll
      for (int b = a; b < 6; ++b) {
        acc[k] = fma(J[a], J[b], acc[k]);
        ++k;
      }
#pragma unroll
    for (int a = 0; a < 6; ++a) acc[21 + a] = fma(J[a], r, acc[21 + a]);
    acc[27] = fma(r, r, acc[27]);
    acc[28] += valid ? 1.0 : 0.0;
  }
  // CTA reduction: warp shuffles, then warp partials through shared memory
  __shared__ double sh[kManifoldThreads / 32][kNE];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kNE; ++k) {
    const double v = warp_sum(acc[k]);
    if (lane == 0) sh[wid][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < kNE) {
    double v = 0.0;
    for (int w = 0; w < kManifoldThreads / 32; ++w) v += sh[w][threadIdx.x];
    partials[blockIdx.x * kNE + threadIdx.x] = v;
  }
}

__global__ void k_reduce_partials(const double* __restrict__ partials, int nblocks,
                                  double* __restrict__ out) {
  // one warp per component, fixed order -> deterministic
  const int k = blockIdx.x;
  double v = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += 32) v += partials[b * kNE + k];
  v = warp_sum(v);
  if (threadIdx.x == 0) out[k] = v;
}

void manifold_device(tlg_model* m, const double R[9], const double t[3], const double* hx,
                     const double* hy, const double* hz, size_t n, double wheel_radius,
                     double lambda_M, double huber, double* r, double* J, uint8_t* valid,
                     double* raw, tlg_normal_eq* ne) {
  tlg_ctx* ctx = m->ctx;
  ensure_grid(m);
  Pose pose;
  for (int i = 0; i < 9; ++i) pose.R[i] = R[i];
  for (int i = 0; i < 3; ++i) pose.t[i] = t[i];
  const unsigned blocks = grid_for(ctx, n, kManifoldThreads, 4);
  double* partials = ctx->ws<double>(S_PARTIALS, static_cast<size_t>(blocks) * kNE + kNE);
  double* out = partials + static_cast<size_t>(blocks) * kNE;
  int* err = ctx->ws<int>(S_FLAGS, 4);
  TLG_CUDA(cudaMemsetAsync(err, 0, sizeof(int), ctx->stream));
  prof_begin(ctx, 0);
  k_manifold<<<blocks, kManifoldThreads, 0, ctx->stream>>>(
      grid_view(m), pose, hx, hy, hz, n, m->kc.r2, m->kc.neg_inv_2s2, m->kc.inv_s2,
      wheel_radius, std::sqrt(lambda_M), huber, r, J, valid, raw, partials, err);
  TLG_LAUNCHED(ctx);
  prof_mark_end(ctx);
  k_reduce_partials<<<kNE, 32, 0, ctx->stream>>>(partials, blocks, out);
  TLG_LAUNCHED(ctx);
  double h[kNE + 1];
  TLG_CUDA(cudaMemcpyAsync(h, out, kNE * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  TLG_CUDA(cudaMemcpyAsync(&h[kNE], err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  TLG_CUDA(cudaStreamSynchronize(ctx->stream));
  prof_collect(ctx);
  int e = 0;
  std::memcpy(&e, &h[kNE], sizeof(int));
  if (e) throw Error(TLG_DOMAIN_ERROR, "non-finite query");
  if (ne) {
    for (int k = 0; k < 21; ++k) ne->A[k] = h[k];
    for (int k = 0; k < 6; ++k) ne->g[k] = h[21 + k];
    ne->cost = h[27];
    ne->valid = h[28];
  }
}

// ---------------------------------------------------------------------------
// moment_feature (terrain_model.cpp:97-107) as CSR: count, scan, fill, sort.
__global__ void k_moment_count(GridView g, const double* __restrict__ x,
                               const double* __restrict__ y, size_t n, double r2,
                               double neg_inv_2b2, uint32_t* __restrict__ cnt,
                               int* __restrict__ err) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double px = x[i], py = y[i];
  if (!isfinite(px) || !isfinite(py)) {
    atomicOr(err, 1);
    cnt[i] = 0;
    return;
  }
  uint32_t c = 0;
  const int qx = static_cast<int>(floor(px / g.cell));
  const int qy = static_cast<int>(floor(py / g.cell));
  const int y_lo = max(qy - g.span - g.gy0, 0), y_hi = min(qy + g.span - g.gy0, g.gny - 1);
  const int x_lo = max(qx - g.span - g.gx0, 0), x_hi = min(qx + g.span - g.gx0, g.gnx - 1);
  if (y_lo <= y_hi)
    for (int gx = x_lo; gx <= x_hi; ++gx) {
      const int b = g.cell_start[gx * g.gny + y_lo], e = g.cell_start[gx * g.gny + y_hi + 1];
      for (int k = b; k < e; ++k) {
        const double d2 = sq2_exact(g.cx[k] - px, g.cy[k] - py);
        if (d2 <= r2 && exp(d2 * neg_inv_2b2) != 0.0) ++c;
      }
    }
  cnt[i] = c;
}

__global__ void k_moment_fill(GridView g, const double* __restrict__ x,
                              const double* __restrict__ y, size_t n, double r2,
                              double neg_inv_2b2, double scale, const uint32_t* __restrict__ rowp,
                              uint32_t* __restrict__ ids, double* __restrict__ vals) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double px = x[i], py = y[i];
  if (!isfinite(px) || !isfinite(py)) return;
  uint32_t o = rowp[i];
  const uint32_t o0 = o;
  const int qx = static_cast<int>(floor(px / g.cell));
  const int qy = static_cast<int>(floor(py / g.cell));
  const int y_lo = max(qy - g.span - g.gy0, 0), y_hi = min(qy + g.span - g.gy0, g.gny - 1);
  const int x_lo = max(qx - g.span - g.gx0, 0), x_hi = min(qx + g.span - g.gx0, g.gnx - 1);
  if (y_lo <= y_hi)
    for (int gx = x_lo; gx <= x_hi; ++gx) {
      const int b = g.cell_start[gx * g.gny + y_lo], e = g.cell_start[gx * g.gny + y_hi + 1];
      for (int k = b; k < e; ++k) {
        const double d2 = sq2_exact(g.cx[k] - px, g.cy[k] - py);
        if (d2 <= r2) {
          const double kv = exp(d2 * neg_inv_2b2);
          if (kv != 0.0) {
            ids[o] = g.id[k];
            vals[o] = scale * kv;
            ++o;
          }
        }
      }
    }
  // ascending ids (SparseVec contract, kernel.hpp:32-34): insertion sort
  for (uint32_t a = o0 + 1; a < o; ++a) {
    const uint32_t ki = ids[a];
    const double kvv = vals[a];
    uint32_t b = a;
    while (b > o0 && ids[b - 1] > ki) {
      ids[b] = ids[b - 1];
      vals[b] = vals[b - 1];
      --b;
    }
    ids[b] = ki;
    vals[b] = kvv;
  }
}

}  // namespace tlg
