// K3 eval_height_grad and K4 manifold_rows_reduce.
//
// K3: predict_height / predict_gradient (terrain_model.cpp:109-143) per
//     query point. Neighbour membership replicates GridIndex2::radius_query
//     (grid_index.hpp:32-48) bit-exactly: same cell coordinates
//     floor(v / cell), same (2*span+1)^2 cell window, same no-FMA
//     r^2 = dx*dx + dy*dy <= cutoff^2 test. Values are FP64 with FMA
//     accumulation (parity: 1e-9 of max(|ref|, sum|w kappa|)).
//
//     Two sweeps:
//     - generic: the reference's 3x3 cell sweep over the CSR centre grid;
//     - lattice (centres are mesh nodes, the select_centers/birth case): a
//       fixed WIN x WIN node window of the dense weight grid W. Pairs are
//       classified once per model (always inside the cutoff disc / boundary /
//       always outside, with 1e-6-cell and 1e-9-radius safety margins), so
//       only boundary pairs run the exact reference test; kappa is separable
//       on the lattice, kappa = e_x(i) e_y(j), and e_x, e_y follow a
//       two-multiply recurrence along the window (two exps per axis); each
//       pair costs two FMAs:
//         S_i = sum_j w_ij e_y(j),  T_i = sum_j w_ij e_y(j) dy_j,
//         z = sum_i e_x(i) S_i, dz/dx = sum_i e_x(i) dx_i S_i / s^2, ...
//       The paper's geometry (and the reference tests') is compiled in, so
//       the class of every pair is a compile-time constant (no per-pair
//       branches, always-outside pairs vanish); other geometries use the
//       same window with runtime class masks.
// K4: the manifold soft-constraint rows (contact.cpp:7-39 +
//     scan_matcher.cpp:221-248), materialised as r / J (column-major rows x 6)
//     / valid, with J^T J, J^T r and the cost reduced in the same pass: each
//     warp drops its 32 rows' 29 products into a shared tile, lane L sums
//     entry L; one partial per CTA, then a fixed-order final reduction
//     (deterministic, no FP64 atomics).
#include <cmath>
#include <math_constants.h>
#include <type_traits>

#include "internal.cuh"

namespace tlg {

struct EvalOut {
  double z, sx, sy;  // sum w k, sum w k (c - x), sum w k (c - y)
  bool sup;
};

// Sweeps the reference's candidate cells of query (x, y); cells of one x
// column are contiguous in cell order, so each column is one index range.
__device__ __forceinline__ EvalOut eval_generic(const GridView& g, double x, double y, double r2,
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

template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

constexpr int ctz32(uint32_t v) {
  int n = 0;
  while (v && !(v & 1u)) {
    v >>= 1;
    ++n;
  }
  return n;
}

// Boundary pair: the exact reference test d2 = fl(dx^2 + dy^2) <= r2 selects
// the weight (a select measured faster than predicated inline-PTX FMAs, which
// block ptxas scheduling: 0.68 vs 0.59 ms)
__device__ __forceinline__ void bd_pair(double& S, double& T, double d2, double r2, double w,
                                        double ey, double eyd) {
  const double wm = d2 <= r2 ? w : 0.0;
  S = fma(wm, ey, S);
  T = fma(wm, eyd, T);
}

// LOOSE (compiled geometries only, dispatched when LatticeView::loose_ok):
// boundary pairs are summed without the cutoff test. A pair that fails it
// lies beyond the cutoff, where kappa_sigma <= exp(-r2 / (2 sigma^2)) (6.8e-15
// with the paper's parameters), so the sum moves by at most
// n_bd kappa(cutoff) |w|max (z) and that times cutoff / sigma^2 (gradient).
// k_cell_flags proves, per lattice cell, that this stays under 1e-10 of a
// lower bound of the parity scales sum |w kappa| and sum |w kappa| d / s^2
// over every point of the cell (10x inside the 1e-9 tolerance); cells that
// fail (weights near zero around them, support fringe) take the exact path.
// Everything else (window, support flag, always-inside/outside pairs) is the
// exact path's.
template <int WIN, int G, bool LOOSE = false>
__device__ __forceinline__ EvalOut eval_lattice(const LatticeView& L, double x, double y,
                                                double r2, double neg_inv_2b2) {
  EvalOut o{0.0, 0.0, 0.0, false};
  const int ib = static_cast<int>(floor((x - L.org_x) * L.inv_res));
  const int jb = static_cast<int>(floor((y - L.org_y) * L.inv_res));
  const int i0 = ib - L.lo, j0 = jb - L.lo;
  // the whole window lies in the zero padding (or beyond): no centre within
  // the cutoff -> unsupported, exactly like an empty radius query
  if (i0 < 0 || j0 < 0 || i0 + WIN > L.ni || j0 + WIN > L.nj) return o;
  // LOOSE: the per-cell flags (k_cell_flags, rebuilt lazily after weight
  // changes) say whether the skipped boundary tests are provably negligible
  // for every point of this cell (bit 1) and whether its four corner nodes
  // are present, which makes every point of the cell supported (bit 0)
  uint32_t cflag = 0;
  if constexpr (LOOSE) {
    cflag = __ldg(L.cflag + static_cast<size_t>(ib) * L.nj + jb);
    if (!(cflag & 2u)) return eval_lattice<WIN, G, false>(L, x, y, r2, neg_inv_2b2);
  }
  // reference hash cells of the point (a division each): only the exact
  // path's boundary tests and the rare support scan below need them
  int qx = 0, qy = 0;
  if constexpr (!LOOSE) {
    qx = static_cast<int>(floor(x / L.cell));
    qy = static_cast<int>(floor(y / L.cell));
  }

  // Row factors. dy^2 is kept exact for the boundary tests; e_y follows the
  // lattice recurrence e(l+1) = e(l) p(l), p(l+1) = p(l) exp(2 c res^2)
  // (c = -1/(2 s^2)), two exps per axis instead of WIN.
  // dy2 carries the reference's cell-window test too: a row outside the
  // (2 span + 1)^2 cell sweep gets dy2 = +inf, so its boundary tests fail
  // without a per-pair predicate (inside pairs never need it, by their margin).
  // Node coordinates are recomputed exactly as k_lattice_axes built them
  // (fl(min + fl(index * res))) instead of loaded: the L1 data path, not the
  // FP64 pipe, binds this kernel. The cell sweep becomes one index range per
  // axis (cells are monotone in the node index).
  int2 rx = make_int2(0, 0), ry = make_int2(0, 0);
  if constexpr (!LOOSE) {
    rx = __ldg(L.xr + min(max(qx - L.xr_base, 0), L.xr_n - 1));
    ry = __ldg(L.yr + min(max(qy - L.yr_base, 0), L.yr_n - 1));
  }
  auto node_x = [&](int i) {
    return __dadd_rn(L.min_x, __dmul_rn(static_cast<double>(i + L.i_org), L.res));
  };
  auto node_y = [&](int j) {
    return __dadd_rn(L.min_y, __dmul_rn(static_cast<double>(j + L.j_org), L.res));
  };
  double ey[WIN], eyd[WIN], dy2[WIN];
  // LOOSE uses no exact pair test, so offsets may drift by an ulp: dy_l =
  // dy_0 + l res (one FMA) instead of the exact node coordinate
  const double dy0 = __dsub_rn(node_y(j0), y);
#pragma unroll
  for (int l = 0; l < WIN; ++l) {
    const int jj = j0 + l;
    const double dy = l == 0 ? dy0 : (LOOSE ? fma(static_cast<double>(l), L.res, dy0)
                                            : __dsub_rn(node_y(jj), y));
    dy2[l] = (jj >= ry.x && jj < ry.y) ? __dmul_rn(dy, dy) : CUDART_INF;
    eyd[l] = dy;
  }
  // compiled geometries are only dispatched when the recurrence is safe
  // (sweep_kind), so their code carries no per-node exp fallback
  constexpr bool kRecAlways = G >= 0;
  const bool rec = kRecAlways || L.rec_ok;
  // LOOSE compiled path: the leading factors of both axes share one exp,
  // exp(c (dx_0^2 + dy_0^2)), applied to z and the gradient sums at the end;
  // the axis chains then start at 1 (exponents stay within ~+-80 there)
#ifndef TLG_SHARED_EXP
#define TLG_SHARED_EXP 1
#endif
  constexpr bool kShared = LOOSE && G >= 0 && TLG_SHARED_EXP;
  const double dx_first = __dsub_rn(node_x(i0), x);
  double common = 1.0;
  if constexpr (kShared) common = exp(fma(dx_first, dx_first, __dmul_rn(eyd[0], eyd[0])) * neg_inv_2b2);
  if (rec) {
    double e = kShared ? 1.0 : exp(__dmul_rn(eyd[0], eyd[0]) * neg_inv_2b2);
    double p = exp(L.c_res * fma(2.0, eyd[0], L.res));
#pragma unroll
    for (int l = 0; l < WIN; ++l) {
      ey[l] = e;
      e *= p;
      p *= L.k2;
    }
  } else if constexpr (!kRecAlways) {
#pragma unroll
    for (int l = 0; l < WIN; ++l) ey[l] = exp(__dmul_rn(eyd[l], eyd[l]) * neg_inv_2b2);
  }
#pragma unroll
  for (int l = 0; l < WIN; ++l) eyd[l] *= ey[l];
  const size_t bidx = static_cast<size_t>(i0) * L.nj + j0;
  // compiled geometries read the window in 16-byte pairs: an odd base is
  // served from the one-element-shifted copy W1 (the pitch nj is even)
  const double* wbase = (G >= 0 && (bidx & 1)) ? L.W1 + bidx + 1 : L.W + bidx;
  double ex_e = 0.0, ex_p = 0.0;
  if (rec) {
    ex_e = kShared ? 1.0 : exp(__dmul_rn(dx_first, dx_first) * neg_inv_2b2);
    ex_p = exp(L.c_res * fma(2.0, dx_first, L.res));
  }
  auto column = [&](auto KC) {
    constexpr int k = decltype(KC)::value;
    const double dx = k == 0 ? dx_first
                             : (LOOSE ? fma(static_cast<double>(k), L.res, dx_first)
                                      : __dsub_rn(node_x(i0 + k), x));
    const double dxx = __dmul_rn(dx, dx);
    const double dx2 = (i0 + k >= rx.x && i0 + k < rx.y) ? dxx : CUDART_INF;  // see dy2
    const double* wc = wbase + static_cast<size_t>(k) * L.nj;
    double S = 0.0, T = 0.0;
    bool any;
    if constexpr (G >= 0) {
      // compiled geometry: always-outside pairs vanish, always-inside pairs
      // carry no test, only boundary pairs run the exact reference test;
      // weights arrive two rows per 16-byte load
      constexpr uint32_t im = kGeoms[G].in[k], bm = kGeoms[G].bd[k];
      constexpr uint32_t need = im | bm;
      static_for<0, (WIN + 1) / 2>([&](auto PC) {
        constexpr int pr = decltype(PC)::value;
        constexpr uint32_t pm = (need >> (2 * pr)) & 3u;
        if constexpr (pm != 0) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(wc) + pr);
          static_for<0, 2>([&](auto HC) {
            constexpr int l = 2 * pr + decltype(HC)::value;
            if constexpr (l < WIN) {
              const double wv = decltype(HC)::value ? v.y : v.x;
              if constexpr (LOOSE && ((need >> l) & 1u)) {
                // every window pair unconditional: the chain starts with a
                // multiply (no zero-initialised accumulator)
                if constexpr (l == ctz32(need)) {
                  S = wv * ey[l];
                  T = wv * eyd[l];
                } else {
                  S = fma(wv, ey[l], S);
                  T = fma(wv, eyd[l], T);
                }
              } else if constexpr ((im >> l) & 1u) {
                S = fma(wv, ey[l], S);
                T = fma(wv, eyd[l], T);
              } else if constexpr ((bm >> l) & 1u) {
                bd_pair(S, T, __dadd_rn(dx2, dy2[l]), r2, wv, ey[l], eyd[l]);
              }
            }
          });
        }
      });
      any = need != 0;
    } else {
      const uint32_t im = L.inmask[k], bm = L.bdmask[k];
#pragma unroll
      for (int l = 0; l < WIN; ++l) {
        if ((im >> l) & 1u) {
          const double w = __ldg(wc + l);
          S = fma(w, ey[l], S);
          T = fma(w, eyd[l], T);
        } else if ((bm >> l) & 1u) {
          if (__dadd_rn(dx2, dy2[l]) <= r2) {
            const double w = __ldg(wc + l);
            S = fma(w, ey[l], S);
            T = fma(w, eyd[l], T);
          }
        }
      }
      any = (im | bm) != 0;
    }
    double ex = ex_e;
    if (rec) {
      ex_e *= ex_p;
      ex_p *= L.k2;
    } else if constexpr (!kRecAlways) {
      ex = exp(dxx * neg_inv_2b2);
    }
    if (any) {
      o.z = fma(ex, S, o.z);
      o.sx = fma(ex * dx, S, o.sx);
      o.sy = fma(ex, T, o.sy);
    }
  };
  static_for<0, WIN>(column);
  if constexpr (kShared) {
    o.z *= common;
    o.sx *= common;
    o.sy *= common;
  }
  // supported: some *present* centre passes the reference test. The cell's
  // four corner nodes are always inside; otherwise scan the window (rare).
  bool sup = false;
  if constexpr (LOOSE) {
    sup = (cflag & 1u) != 0;
  } else if (L.corner_ok) {
    const int* pc = L.P + static_cast<size_t>(ib) * L.nj + jb;
    sup = (__ldg(pc) | __ldg(pc + 1) | __ldg(pc + L.nj) | __ldg(pc + L.nj + 1)) != 0;
  }
  if (!sup) {
    if constexpr (LOOSE) {
      qx = static_cast<int>(floor(x / L.cell));
      qy = static_cast<int>(floor(y / L.cell));
    }
    for (int k = 0; k < WIN && !sup; ++k) {
      const AxisNode ak = L.ax[i0 + k];
      const double dx = __dsub_rn(ak.c, x);
      const double dx2 = __dmul_rn(dx, dx);
      const bool colok = abs(ak.cell - qx) <= L.span;
      const int* pc = L.P + static_cast<size_t>(i0 + k) * L.nj + j0;
      for (int l = 0; l < WIN; ++l) {
        const AxisNode al = L.ay[j0 + l];
        const double dy = __dsub_rn(al.c, y);
        const bool in = ((L.inmask[k] >> l) & 1u) ||
                        (((L.bdmask[k] >> l) & 1u) && colok && abs(al.cell - qy) <= L.span &&
                         __dadd_rn(dx2, __dmul_rn(dy, dy)) <= r2);
        if (in && __ldg(pc + l)) {
          sup = true;
          break;
        }
      }
    }
  }
  o.sup = sup;
  return o;
}

// KIND: 0 = generic sweep, 1..kMaxWin = lattice window with runtime pair
// classes, 100 + g = lattice window of compiled geometry kGeoms[g].
template <int KIND>
__device__ __forceinline__ EvalOut eval_any(const GridView& g, const LatticeView& L, double x,
                                            double y, double r2, double neg_inv_2b2) {
  if constexpr (KIND == 0)
    return eval_generic(g, x, y, r2, neg_inv_2b2);
  else if constexpr (KIND >= 100)
    return eval_lattice<kGeoms[(KIND - 100) % 100].win, (KIND - 100) % 100, (KIND >= 200)>(
        L, x, y, r2, neg_inv_2b2);
  else
    return eval_lattice<KIND, -1>(L, x, y, r2, neg_inv_2b2);
}

template <int KIND>
#ifndef TLG_EVAL_THREADS
#define TLG_EVAL_THREADS 256
#endif
#ifndef TLG_EVAL_MINB
#define TLG_EVAL_MINB 2
#endif
__global__ void __launch_bounds__(TLG_EVAL_THREADS, TLG_EVAL_MINB) k_eval(GridView g, LatticeView L,
                                                 const double* __restrict__ x,
                                                 const double* __restrict__ y, size_t n,
                                                 double r2, double neg_inv_2s2, double inv_s2,
                                                 double* __restrict__ z,
                                                 uint8_t* __restrict__ sup,
                                                 double* __restrict__ gx,
                                                 double* __restrict__ gy, int* __restrict__ err) {
  // Same schedule as k_manifold: warps claim chunks of 8 rows-of-32 (err[2..3]
  // is the counter), the next row's query is loaded one iteration ahead.
  constexpr unsigned long long kChunk = 8;
  const int lane = threadIdx.x & 31;
  const size_t witer = (n + 31) / 32;
  auto claim = [&]() {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(reinterpret_cast<unsigned long long*>(err + 2), kChunk);
    return __shfl_sync(0xffffffffu, c, 0);
  };
  unsigned long long chunk = claim();
  if (chunk >= witer) return;
  unsigned long long next = claim();
  size_t base = static_cast<size_t>(chunk) * 32;
  size_t b_end = std::min(n, static_cast<size_t>((chunk + kChunk) * 32));
  double px = 0.0, py = 0.0;
  if (base + lane < n) {
    px = x[base + lane];
    py = y[base + lane];
  }
  for (;;) {
    const size_t i = base + lane;
    size_t pf = base + 32 < b_end ? base + 32 : (next < witer ? static_cast<size_t>(next) * 32 : n);
    pf += lane;
    double nx = 0.0, ny = 0.0;
    if (pf < n) {
      nx = x[pf];
      ny = y[pf];
    }
    if (i < n) {
      if (!isfinite(px) || !isfinite(py)) {
        atomicOr(err, 1);
      } else {
        const EvalOut o = eval_any<KIND>(g, L, px, py, r2, neg_inv_2s2);
        if (z) z[i] = o.sup ? o.z : 0.0;
        if (sup) sup[i] = o.sup ? 1 : 0;
        if (gx) gx[i] = o.sx * inv_s2;
        if (gy) gy[i] = o.sy * inv_s2;
      }
    }
    px = nx;
    py = ny;
    base += 32;
    if (base >= b_end) {
      if (next >= witer) break;
      chunk = next;
      next = claim();
      base = static_cast<size_t>(chunk) * 32;
      b_end = std::min(n, static_cast<size_t>((chunk + kChunk) * 32));
    }
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

int sweep_kind(const tlg_model* m) {
  if (!m->lat.valid) return 0;
  const LatticeView v = lattice_view(m);
  if (m->lat.geom_id < 0 || !v.rec_ok) return m->lat.win;
  return (v.loose_ok && !m->exact_cutoff ? 200 : 100) + m->lat.geom_id;
}

#define TLG_KIND_DISPATCH(KINDV, CALL)                   \
  switch (KINDV) {                                       \
    case 100: { constexpr int W_ = 100; CALL; } break;   \
    case 101: { constexpr int W_ = 101; CALL; } break;   \
    case 200: { constexpr int W_ = 200; CALL; } break;   \
    case 201: { constexpr int W_ = 201; CALL; } break;   \
    case 4: { constexpr int W_ = 4; CALL; } break;       \
    case 5: { constexpr int W_ = 5; CALL; } break;       \
    case 6: { constexpr int W_ = 6; CALL; } break;       \
    case 7: { constexpr int W_ = 7; CALL; } break;       \
    case 8: { constexpr int W_ = 8; CALL; } break;       \
    case 9: { constexpr int W_ = 9; CALL; } break;       \
    case 10: { constexpr int W_ = 10; CALL; } break;     \
    case 11: { constexpr int W_ = 11; CALL; } break;     \
    case 12: { constexpr int W_ = 12; CALL; } break;     \
    case 13: { constexpr int W_ = 13; CALL; } break;     \
    case 14: { constexpr int W_ = 14; CALL; } break;     \
    default: { constexpr int W_ = 0; CALL; } break;      \
  }

void eval_device(tlg_model* m, const double* x, const double* y, size_t n, double* z,
                 uint8_t* sup, double* gx, double* gy) {
  tlg_ctx* ctx = m->ctx;
  ensure_grid(m);
  int* err = ctx->ws<int>(S_FLAGS, 4);
  TLG_CUDA(cudaMemsetAsync(err, 0, 4 * sizeof(int), ctx->stream));
  if (n) {
    const GridView g = grid_view(m);
    const int kind = prepare_sweep(m);
    const LatticeView L = lattice_view(m);
    prof_begin(ctx, 1);
    TLG_KIND_DISPATCH(kind,
                      (k_eval<W_><<<grid_for(ctx, n, TLG_EVAL_THREADS, TLG_EVAL_MINB), TLG_EVAL_THREADS, 0,
                                 ctx->stream>>>(
                          g, L, x, y, n, m->kc.r2, m->kc.neg_inv_2s2, m->kc.inv_s2, z, sup, gx,
                          gy, err)));
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
// one 512-thread CTA per SM (16 warps at 128 registers, the same residency
// as two 256-thread CTAs; measured 1 % faster: 0.399 vs 0.404 ms at C5)
#ifndef TLG_MANIFOLD_THREADS
#define TLG_MANIFOLD_THREADS 512
#endif
#ifndef TLG_MANIFOLD_MINB
#define TLG_MANIFOLD_MINB 1
#endif
constexpr int kManifoldThreads = TLG_MANIFOLD_THREADS;
#ifndef TLG_MANIFOLD_CHUNK
#define TLG_MANIFOLD_CHUNK 8
#endif
constexpr unsigned long long kManifoldChunk = TLG_MANIFOLD_CHUNK;  // warp-iterations per claim

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Index of Gram entry (i, j) of V = [J0..J5, r, valid] in the 29-entry
// normal-equation layout (A upper row-major, g, cost, valid), -1 if unused.
__device__ __forceinline__ int ne_index(int i, int j) {
  if (i <= j && j < 6) return i * 6 - i * (i - 1) / 2 + (j - i);
  if (i < 6 && j == 6) return 21 + i;
  if (i == 6 && j == 6) return 27;
  if (i == 7 && j == 7) return 28;
  return -1;
}

template <int KIND>
__global__ void __launch_bounds__(kManifoldThreads, TLG_MANIFOLD_MINB) k_manifold(
    GridView g, LatticeView L, Pose pose, const double* __restrict__ hx,
    const double* __restrict__ hy, const double* __restrict__ hz, size_t n, double r2,
    double neg_inv_2s2, double inv_s2, double wheel_radius, double sl, double huber,
    double* __restrict__ out_r, double* __restrict__ out_J, uint8_t* __restrict__ out_valid,
    double* __restrict__ out_raw, double* __restrict__ partials, size_t nchunks,
    size_t chunk_base, size_t ldj, int* __restrict__ err) {
  // Normal equations on the FP64 tensor pipe: each point contributes the
  // rank-1 Gram V V^T of V = [J, r, valid] (8 components); a warp stages its
  // 32 rows' V in shared memory and 8 DMMA m8n8k4 steps add V^T V into an
  // 8x8 accumulator held as 2 doubles per lane. Per claimed chunk the 29
  // used entries go to partials[entry][chunk] (fixed slots -> the final
  // reduction is order-fixed and deterministic despite dynamic claiming).
  // V staged transposed, [component][row] with a 36-double pitch: the
  // per-lane stores and the fragment loads are both bank-conflict free
  constexpr int kVP = 36;
  __shared__ __align__(16) double vt[kManifoldThreads / 32][8 * kVP];
  double c0 = 0.0, c1 = 0.0;
  const double* R = pose.R;
  const int lane = threadIdx.x & 31;
  double* V = vt[threadIdx.x >> 5];
  const int gi = lane >> 2, gj0 = 2 * (lane & 3);
  const int e0 = ne_index(gi, gj0), e1 = ne_index(gi, gj0 + 1);
  // Warps claim contiguous chunks of kManifoldChunk rows-of-32 from a global
  // counter: with scan-binned input consecutive iterations hit the same /
  // neighbouring lattice cells, so the weight window stays L1-resident, and
  // dynamic claiming keeps the warps of a CTA finishing together.
  // The lever arms stream from HBM (cold): the next row-of-32's loads are
  // issued one iteration ahead, and the next chunk is claimed one chunk ahead
  // so the prefetch also crosses chunk boundaries.
  const size_t witer = (n + 31) / 32;
  auto claim = [&]() {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(reinterpret_cast<unsigned long long*>(err + 2), kManifoldChunk);
    return __shfl_sync(0xffffffffu, c, 0);
  };
  unsigned long long chunk = claim();
  if (chunk >= witer) return;
  unsigned long long next = claim();
  size_t base = static_cast<size_t>(chunk) * 32;
  size_t b_end = std::min(n, static_cast<size_t>((chunk + kManifoldChunk) * 32));
  double h0 = 0.0, h1 = 0.0, h2 = 0.0;
  if (base + lane < n) {
    h0 = hx[base + lane];
    h1 = hy[base + lane];
    h2 = hz[base + lane];
  }
  for (;;) {
    const size_t i = base + lane;
    const bool live = i < n;
    size_t pf = base + 32 < b_end ? base + 32 : (next < witer ? static_cast<size_t>(next) * 32 : n);
    pf += lane;
    double nh0 = 0.0, nh1 = 0.0, nh2 = 0.0;
    if (pf < n) {
      nh0 = hx[pf];
      nh1 = hy[pf];
      nh2 = hz[pf];
    }
    // xi = R h + t (leg_model.cpp:31, contact.cpp:183)
    const double xi0 = fma(R[2], h2, fma(R[1], h1, R[0] * h0)) + pose.t[0];
    const double xi1 = fma(R[5], h2, fma(R[4], h1, R[3] * h0)) + pose.t[1];
    const double xi2 = fma(R[8], h2, fma(R[7], h1, R[6] * h0)) + pose.t[2];
    double r = 0.0, raw = 0.0, J[6] = {0, 0, 0, 0, 0, 0};
    bool valid = false;
    if (!live) {
    } else if (!isfinite(xi0) || !isfinite(xi1)) {
      atomicOr(err, 1);
    } else {
      const EvalOut o = eval_any<KIND>(g, L, xi0, xi1, r2, neg_inv_2s2);
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
    if (live) {
      if (out_r) out_r[i] = r;
      if (out_raw) out_raw[i] = raw;
      if (out_valid) out_valid[i] = valid ? 1 : 0;
      if (out_J) {
#pragma unroll
        for (int c = 0; c < 6; ++c) out_J[c * ldj + i] = J[c];
      }
    }
#pragma unroll
    for (int c = 0; c < 6; ++c) V[c * kVP + lane] = J[c];
    V[6 * kVP + lane] = r;
    V[7 * kVP + lane] = valid ? 1.0 : 0.0;
    __syncwarp();
#pragma unroll
    for (int st = 0; st < 8; ++st) {
      // A[m][k] = B[k][m] = V_row(4 st + k)[m]; lane holds m = lane >> 2, k = lane & 3
      const double v = V[(lane >> 2) * kVP + 4 * st + (lane & 3)];
      dmma884(c0, c1, v, v);
    }
    __syncwarp();
    h0 = nh0;
    h1 = nh1;
    h2 = nh2;
    base += 32;
    if (base >= b_end) {  // chunk done: flush its Gram, move to the pre-claimed one
      if (e0 >= 0) partials[(size_t)e0 * nchunks + chunk_base + chunk / kManifoldChunk] = c0;
      if (e1 >= 0) partials[(size_t)e1 * nchunks + chunk_base + chunk / kManifoldChunk] = c1;
      c0 = c1 = 0.0;
      if (next >= witer) break;
      chunk = next;
      next = claim();
      base = static_cast<size_t>(chunk) * 32;
      b_end = std::min(n, static_cast<size_t>((chunk + kManifoldChunk) * 32));
    }
  }
}

// Order-fixed reduction of the per-chunk Gram partials, two levels in one
// launch: block (entry, seg) sums a fixed contiguous range of chunks (thread t
// a strided run, then a fixed tree) into seg_part[entry][seg]; the last of an
// entry's kRedSeg blocks to finish (an arrival counter) adds the kRedSeg
// segment sums in order and resets the counter. The result does not depend on
// the arrival order, so it is reproducible run to run; kNE x kRedSeg blocks
// spread the ~9 MB of partials (C5) over the SMs instead of kNE of them.
// Block (0, 0) also appends the non-finite flag, so one D2H copy returns
// everything.
constexpr int kRedThreads = 256;
constexpr int kRedSeg = 8;
__global__ void __launch_bounds__(kRedThreads) k_reduce_chunks(const double* __restrict__ partials,
                                                               size_t nchunks,
                                                               const int* __restrict__ err,
                                                               double* __restrict__ out,
                                                               double* __restrict__ seg_part,
                                                               unsigned* __restrict__ arrive,
                                                               double* __restrict__ host_out) {
  __shared__ double sh[kRedThreads];
  __shared__ bool last;
  const int entry = blockIdx.x / kRedSeg, seg = blockIdx.x % kRedSeg;
  const double* p = partials + (size_t)entry * nchunks;
  const size_t c0 = nchunks * seg / kRedSeg, c1 = nchunks * (seg + 1) / kRedSeg;
  double v = 0.0;
  size_t c = c0 + threadIdx.x;
  for (; c + 7 * kRedThreads < c1; c += 8 * kRedThreads) {
    double q[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) q[u] = p[c + u * kRedThreads];
#pragma unroll
    for (int u = 0; u < 8; ++u) v += q[u];
  }
  for (; c < c1; c += kRedThreads) v += p[c];
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = kRedThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    seg_part[entry * kRedSeg + seg] = sh[0];
    __threadfence();
    last = atomicAdd(arrive + entry, 1u) == kRedSeg - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double s = 0.0;
    for (int k = 0; k < kRedSeg; ++k) s += __ldcg(seg_part + entry * kRedSeg + k);
    out[entry] = s;
    if (host_out) host_out[entry] = s;  // mapped pinned memory: no D2H copy
    arrive[entry] = 0u;  // ready for the next call
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[kNE] = err[0] ? 1.0 : 0.0;
    if (host_out) host_out[kNE] = out[kNE];
  }
}

// Device view of the context's pinned staging buffer (written directly by
// the reduction: one fewer copy-engine round trip per call)
static double* mapped(double* h) {
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, h, 0) == cudaSuccess) return static_cast<double*>(d);
  (void)cudaGetLastError();  // not mapped: fall back to the copy, clear the error
  return nullptr;
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
  const unsigned blocks = grid_for(ctx, n, kManifoldThreads, TLG_MANIFOLD_MINB);
  const size_t nchunks = std::max<size_t>(1, ((n + 31) / 32 + kManifoldChunk - 1) / kManifoldChunk);
  if (n == 0) {  // no chunk is claimed: the (single) partial slot must read as zero
    double* p0 = ctx->ws<double>(S_PARTIALS, nchunks * kNE + 2 * kNE);
    TLG_CUDA(cudaMemsetAsync(p0, 0, nchunks * kNE * sizeof(double), ctx->stream));
  }
  double* partials = ctx->ws<double>(S_PARTIALS, nchunks * kNE + kNE + 1);
  double* out = partials + nchunks * kNE;
  double* seg_part = ctx->ws<double>(S_REDSEG, kNE * kRedSeg);
  // err[0]: non-finite flag; err[2..3]: 64-bit chunk counter (8-byte aligned);
  // err[4..]: the reduction's arrival counters (one memset clears all)
  int* err = ctx->ws<int>(S_FLAGS, 4 + kNE);
  unsigned* arrive = reinterpret_cast<unsigned*>(err + 4);
  double* h = static_cast<double*>(ctx->host_stage((kNE + 1) * sizeof(double)));  // pinned
  TLG_CUDA(cudaMemsetAsync(err, 0, (4 + kNE) * sizeof(int), ctx->stream));
  const GridView g = grid_view(m);
  const int kind = prepare_sweep(m);
  const LatticeView L = lattice_view(m);
  const double sl = std::sqrt(lambda_M);
  prof_begin(ctx, 0);
  TLG_KIND_DISPATCH(kind,
                    (k_manifold<W_><<<blocks, kManifoldThreads, 0, ctx->stream>>>(
                        g, L, pose, hx, hy, hz, n, m->kc.r2, m->kc.neg_inv_2s2, m->kc.inv_s2,
                        wheel_radius, sl, huber, r, J, valid, raw, partials, nchunks, 0, n,
                        err)));
  TLG_LAUNCHED(ctx);
  prof_mark_end(ctx);
  double* hd = mapped(h);
  k_reduce_chunks<<<kNE * kRedSeg, kRedThreads, 0, ctx->stream>>>(partials, nchunks, err, out,
                                                                   seg_part, arrive, hd);
  TLG_LAUNCHED(ctx);
  if (!hd) TLG_CUDA(cudaMemcpyAsync(h, out, (kNE + 1) * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  TLG_CUDA(cudaStreamSynchronize(ctx->stream));
  prof_collect(ctx);
  if (h[kNE] != 0.0) throw Error(TLG_DOMAIN_ERROR, "non-finite query");
  if (ne) {
    for (int k = 0; k < 21; ++k) ne->A[k] = h[k];
    for (int k = 0; k < 6; ++k) ne->g[k] = h[21 + k];
    ne->cost = h[27];
    ne->valid = h[28];
  }
}

// Host-resident lever arms: the H2D copy of slice s+1 (copy stream) overlaps
// the kernel on slice s (compute stream); every slice is a whole number of
// 8-iteration chunks, so the per-chunk partials of all slices form one
// order-fixed reduction, exactly as in a single launch.
void manifold_device_streamed(tlg_model* m, const double R[9], const double t[3],
                              const double* hx, const double* hy, const double* hz, size_t n,
                              double wheel_radius, double lambda_M, double huber, double* r,
                              double* J, uint8_t* valid, double* raw, tlg_normal_eq* ne) {
  tlg_ctx* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  ensure_grid(m);
  if (!ctx->copy_stream) {
    TLG_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    for (auto& e : ctx->copy_ev) TLG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  Pose pose;
  for (int i = 0; i < 9; ++i) pose.R[i] = R[i];
  for (int i = 0; i < 3; ++i) pose.t[i] = t[i];
  const size_t nchunks = std::max<size_t>(1, ((n + 31) / 32 + kManifoldChunk - 1) / kManifoldChunk);
  double* partials = ctx->ws<double>(S_PARTIALS, nchunks * kNE + kNE + 1);
  double* out = partials + nchunks * kNE;
  double* seg_part = ctx->ws<double>(S_REDSEG, kNE * kRedSeg);
  int* err = ctx->ws<int>(S_FLAGS, 4 + kNE);
  unsigned* arrive = reinterpret_cast<unsigned*>(err + 4);
  double* h = static_cast<double*>(ctx->host_stage((kNE + 1) * sizeof(double)));
  double* dx = ctx->ws<double>(S_IN_HX, n);
  double* dy = ctx->ws<double>(S_IN_HY, n);
  double* dz = ctx->ws<double>(S_IN_HZ, n);
  TLG_CUDA(cudaMemsetAsync(err, 0, (4 + kNE) * sizeof(int), s));
  const GridView g = grid_view(m);
  const int kind = prepare_sweep(m);
  const LatticeView L = lattice_view(m);
  const double sl = std::sqrt(lambda_M);
  constexpr size_t kRowsPerChunk = 32 * kManifoldChunk;
  constexpr int kSlices = 8;
  const size_t slice = ((n + kSlices - 1) / kSlices + kRowsPerChunk - 1) / kRowsPerChunk * kRowsPerChunk;
  // the compute stream must not overtake earlier users of the input slots
  TLG_CUDA(cudaEventRecord(ctx->copy_ev[kSlices], s));
  TLG_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->copy_ev[kSlices], 0));
  int si = 0;
  for (size_t off = 0; off < n; off += slice, ++si) {
    const size_t nc = std::min(slice, n - off);
    TLG_CUDA(cudaMemcpyAsync(dx + off, hx + off, nc * 8, cudaMemcpyHostToDevice, ctx->copy_stream));
    TLG_CUDA(cudaMemcpyAsync(dy + off, hy + off, nc * 8, cudaMemcpyHostToDevice, ctx->copy_stream));
    TLG_CUDA(cudaMemcpyAsync(dz + off, hz + off, nc * 8, cudaMemcpyHostToDevice, ctx->copy_stream));
    TLG_CUDA(cudaEventRecord(ctx->copy_ev[si], ctx->copy_stream));
    TLG_CUDA(cudaStreamWaitEvent(s, ctx->copy_ev[si], 0));
    TLG_CUDA(cudaMemsetAsync(err + 2, 0, 2 * sizeof(int), s));
    const unsigned blocks = grid_for(ctx, nc, kManifoldThreads, TLG_MANIFOLD_MINB);
    TLG_KIND_DISPATCH(kind,
                      (k_manifold<W_><<<blocks, kManifoldThreads, 0, s>>>(
                          g, L, pose, dx + off, dy + off, dz + off, nc, m->kc.r2,
                          m->kc.neg_inv_2s2, m->kc.inv_s2, wheel_radius, sl, huber,
                          r ? r + off : nullptr, J ? J + off : nullptr,
                          valid ? valid + off : nullptr, raw ? raw + off : nullptr, partials,
                          nchunks, off / kRowsPerChunk, n, err)));
    TLG_LAUNCHED(ctx);
  }
  double* hd = mapped(h);
  k_reduce_chunks<<<kNE * kRedSeg, kRedThreads, 0, s>>>(partials, nchunks, err, out, seg_part,
                                                         arrive, hd);
  TLG_LAUNCHED(ctx);
  if (!hd) TLG_CUDA(cudaMemcpyAsync(h, out, (kNE + 1) * sizeof(double), cudaMemcpyDeviceToHost, s));
  TLG_CUDA(cudaStreamSynchronize(s));
  if (h[kNE] != 0.0) throw Error(TLG_DOMAIN_ERROR, "non-finite query");
  if (ne) {
    for (int k = 0; k < 21; ++k) ne->A[k] = h[k];
    for (int k = 0; k < 6; ++k) ne->g[k] = h[21 + k];
    ne->cost = h[27];
    ne->valid = h[28];
  }
}

}  // namespace tlg
