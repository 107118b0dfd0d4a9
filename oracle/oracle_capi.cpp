// TEST INFRASTRUCTURE — C entry points over the CPU oracle, loaded by
// tests/ (ctypes) and bench.py's cpu_baseline leg only. Status codes mirror
// include/terralio_gpu.h so tests can compare error behaviour 1:1.
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "terralio_oracle.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;

enum {
  ORC_OK = 0,
  ORC_INVALID_ARGUMENT = 1,
  ORC_DOMAIN_ERROR = 2,
  ORC_NO_SUPPORTED_CENTERS = 3,
  ORC_RUNTIME_ERROR = 4,
  ORC_BUFFER_TOO_SMALL = 7,
};

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return ORC_OK;
  } catch (const NoSupportedCenters& e) {
    g_err = e.what();
    return ORC_NO_SUPPORTED_CENTERS;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return ORC_INVALID_ARGUMENT;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return ORC_DOMAIN_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ORC_RUNTIME_ERROR;
  }
}

struct KP {
  double sigma, sigma_eps, lambda, cutoff_radius;
};
struct CP {
  double mesh_resolution, accept_radius;
  int accept_count;
  int pad;
  double roi_min_x, roi_min_y, roi_max_x, roi_max_y;
};

KernelParams to_kp(const KP* k) {
  KernelParams p;
  p.sigma = k->sigma;
  p.sigma_eps = k->sigma_eps;
  p.lambda = k->lambda;
  p.cutoff_radius = k->cutoff_radius;
  return p;
}
CenterSet to_cs(const CP* c, const double* cx, const double* cy, size_t n) {
  CenterSet s;
  s.mesh_resolution = c->mesh_resolution;
  s.accept_radius = c->accept_radius;
  s.accept_count = c->accept_count;
  s.roi = {{c->roi_min_x, c->roi_min_y}, {c->roi_max_x, c->roi_max_y}};
  s.centers.resize(n);
  for (size_t i = 0; i < n; ++i) s.centers[i] = {cx[i], cy[i]};
  return s;
}
TerrainObservation to_obs(const double* x, const double* y, const double* z, size_t m) {
  TerrainObservation o;
  o.xy.resize(m);
  o.z.assign(z, z + m);
  for (size_t i = 0; i < m; ++i) o.xy[i] = {x[i], y[i]};
  return o;
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

// ---- RNG: std::mt19937_64 with libstdc++ distributions ----------------------
void* orc_rng_new(unsigned long long seed) { return new std::mt19937_64(seed); }
void orc_rng_free(void* r) { delete static_cast<std::mt19937_64*>(r); }
void orc_uniform(void* r, double lo, double hi, size_t n, double* out) {
  std::uniform_real_distribution<double> u(lo, hi);
  auto& g = *static_cast<std::mt19937_64*>(r);
  for (size_t i = 0; i < n; ++i) out[i] = u(g);
}
int orc_uniform_int(void* r, int lo, int hi) {
  std::uniform_int_distribution<int> u(lo, hi);
  return u(*static_cast<std::mt19937_64*>(r));
}
void* orc_normal_new(double mean, double sd) { return new std::normal_distribution<double>(mean, sd); }
void orc_normal_free(void* d) { delete static_cast<std::normal_distribution<double>*>(d); }
void orc_normal(void* d, void* r, size_t n, double* out) {
  auto& nd = *static_cast<std::normal_distribution<double>*>(d);
  auto& g = *static_cast<std::mt19937_64*>(r);
  for (size_t i = 0; i < n; ++i) out[i] = nd(g);
}

// ---- kernel.cpp --------------------------------------------------------------
int orc_kernel_finalize(KP* k) {
  return guarded([&] {
    KernelParams p = to_kp(k);
    p.finalize();
    k->cutoff_radius = p.cutoff_radius;
  });
}
int orc_kernel_eval(const KP* k, double xx, double xy, double cx, double cy, double bw,
                    double* out) {
  return guarded([&] { *out = kernel_eval(to_kp(k), {xx, xy}, {cx, cy}, bw); });
}
double orc_sigma_tilde(const KP* k) { return to_kp(k).sigma_tilde(); }
double orc_moment_scale(const KP* k) { return to_kp(k).moment_scale(); }

// ---- grid_index.hpp ------------------------------------------------------------
void* orc_grid_new(double cell, const double* x, const double* y, size_t n) {
  auto* g = new GridIndex2(cell);
  for (size_t i = 0; i < n; ++i) g->insert({x[i], y[i]});
  return g;
}
void orc_grid_free(void* g) { delete static_cast<GridIndex2*>(g); }
size_t orc_grid_query(void* g, double qx, double qy, double r, unsigned* out, size_t cap) {
  const auto ids = static_cast<GridIndex2*>(g)->radius_query({qx, qy}, r);
  for (size_t i = 0; i < ids.size() && i < cap; ++i) out[i] = ids[i];
  return ids.size();
}

// ---- center_select.cpp ---------------------------------------------------------
int orc_supported_mesh_nodes(const double* x, const double* y, const double* z, size_t m,
                             size_t zn, double rminx, double rminy, double rmaxx,
                             double rmaxy, double res, double r_a, int count, int throw_empty,
                             double* out_x, double* out_y, size_t cap, size_t* out_n) {
  return guarded([&] {
    TerrainObservation o;
    o.xy.resize(m);
    for (size_t i = 0; i < m; ++i) o.xy[i] = {x[i], y[i]};
    o.z.assign(z, z + zn);
    const Rect roi{{rminx, rminy}, {rmaxx, rmaxy}};
    std::vector<V2> nodes = throw_empty ? select_centers(o, roi, res, r_a, count).centers
                                        : supported_mesh_nodes(o, roi, res, r_a, count);
    *out_n = nodes.size();
    if (nodes.size() > cap) throw std::length_error("buffer too small");
    for (size_t i = 0; i < nodes.size(); ++i) {
      out_x[i] = nodes[i].x;
      out_y[i] = nodes[i].y;
    }
  });
}

// ---- TerrainModel ----------------------------------------------------------------
int orc_model_new(const KP* k, const CP* c, const double* cx, const double* cy, size_t n,
                  void** out) {
  return guarded([&] { *out = new TerrainModel(to_kp(k), to_cs(c, cx, cy, n)); });
}
void orc_model_free(void* m) { delete static_cast<TerrainModel*>(m); }
size_t orc_model_num_centers(void* m) { return static_cast<TerrainModel*>(m)->num_centers(); }
size_t orc_model_num_blocks(void* m) { return static_cast<TerrainModel*>(m)->num_blocks(); }
void orc_model_kernel(void* m, KP* k) {
  const auto& p = static_cast<TerrainModel*>(m)->kernel();
  *k = {p.sigma, p.sigma_eps, p.lambda, p.cutoff_radius};
}
void orc_model_centers(void* m, double* cx, double* cy) {
  const auto& c = static_cast<TerrainModel*>(m)->centers().centers;
  for (size_t i = 0; i < c.size(); ++i) {
    cx[i] = c[i].x;
    cy[i] = c[i].y;
  }
}
void orc_model_weights(void* m, double* w) {
  const auto& v = static_cast<TerrainModel*>(m)->weights();
  std::memcpy(w, v.data(), v.size() * sizeof(double));
}
void orc_model_set_weights(void* m, const double* w) {
  auto* t = static_cast<TerrainModel*>(m);
  t->set_weights(std::vector<double>(w, w + t->num_centers()));
}
void orc_model_block_index(void* m, unsigned* out) {
  auto* t = static_cast<TerrainModel*>(m);
  for (size_t i = 0; i < t->num_centers(); ++i) out[i] = t->block_of(static_cast<unsigned>(i));
}
size_t orc_model_block_size(void* m, unsigned b) {
  return static_cast<TerrainModel*>(m)->block_members(b).size();
}
void orc_model_block_members(void* m, unsigned b, unsigned* out) {
  const auto& v = static_cast<TerrainModel*>(m)->block_members(b);
  for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
}
// column-major bn x bn
void orc_model_block_info_inverse(void* m, unsigned b, double* out) {
  const Mat& a = static_cast<TerrainModel*>(m)->block_info_inverse(b);
  std::memcpy(out, a.a.data(), a.a.size() * sizeof(double));
}

// Batch predict over points, parallel over points with `threads` workers
// (concurrent readers are allowed). Any output may be NULL.
int orc_model_predict(void* m, const double* x, const double* y, size_t n, double* z,
                      unsigned char* sup, double* gx, double* gy, int threads) {
  auto* t = static_cast<TerrainModel*>(m);
  return guarded([&] {
    auto work = [&](size_t b, size_t e) {
      for (size_t i = b; i < e; ++i) {
        if (z || sup) {
          const HeightQuery q = t->predict_height({x[i], y[i]});
          if (z) z[i] = q.z;
          if (sup) sup[i] = q.supported ? 1 : 0;
        }
        if (gx || gy) {
          const V2 g = t->predict_gradient({x[i], y[i]});
          if (gx) gx[i] = g.x;
          if (gy) gy[i] = g.y;
        }
      }
    };
    if (threads <= 1) {
      work(0, n);
      return;
    }
    std::vector<std::thread> pool;
    const size_t chunk = (n + threads - 1) / threads;
    for (int w = 0; w < threads; ++w) {
      const size_t b = w * chunk, e = std::min(n, b + chunk);
      if (b < e) pool.emplace_back(work, b, e);
    }
    for (auto& th : pool) th.join();
  });
}

// Parity scales of the height and gradient at each point:
// s = sum |w_i kappa_sigma(x, c_i)|, g = sum |w_i kappa_sigma| d_i / sigma^2
// over the reference's neighbour set (test infrastructure).
int orc_model_scales(void* m, const double* x, const double* y, size_t n, double* s, double* g,
                     int threads) {
  auto* t = static_cast<TerrainModel*>(m);
  return guarded([&] {
    const double sig = t->kernel().sigma, cut = t->kernel().cutoff_radius;
    const auto& w = t->weights();
    const auto& c = t->centers().centers;
    auto work = [&](size_t b, size_t e) {
      for (size_t i = b; i < e; ++i) {
        double a = 0.0, q = 0.0;
        for (unsigned id : t->centers_near({x[i], y[i]}, cut)) {
          const double dx = x[i] - c[id].x, dy = y[i] - c[id].y;
          const double d2 = dx * dx + dy * dy;
          const double v = std::abs(w[id] * std::exp(-d2 / (2.0 * sig * sig)));
          a += v;
          q += v * std::sqrt(d2) / (sig * sig);
        }
        s[i] = a;
        g[i] = q;
      }
    };
    std::vector<std::thread> pool;
    const int nt = std::max(1, threads);
    const size_t chunk = (n + nt - 1) / nt;
    for (int k = 0; k < nt; ++k) {
      const size_t b = k * chunk, e = std::min(n, b + chunk);
      if (b < e) pool.emplace_back(work, b, e);
    }
    for (auto& th : pool) th.join();
  });
}

size_t orc_model_centers_near(void* m, double qx, double qy, unsigned* out, size_t cap) {
  auto* t = static_cast<TerrainModel*>(m);
  const auto ids = t->centers_near({qx, qy}, t->kernel().cutoff_radius);
  for (size_t i = 0; i < ids.size() && i < cap; ++i) out[i] = ids[i];
  return ids.size();
}

int orc_model_moment_feature(void* m, double qx, double qy, unsigned* ids, double* vals,
                             size_t cap, size_t* out_n) {
  return guarded([&] {
    const SparseVec f = static_cast<TerrainModel*>(m)->moment_feature({qx, qy});
    *out_n = f.entries.size();
    for (size_t i = 0; i < f.entries.size() && i < cap; ++i) {
      ids[i] = f.entries[i].first;
      vals[i] = f.entries[i].second;
    }
  });
}

int orc_model_recursive_update(void* m, const double* x, const double* y, const double* z,
                               size_t mm, size_t zn, int allow_birth, unsigned long long* rep) {
  return guarded([&] {
    TerrainObservation o;
    o.xy.resize(mm);
    for (size_t i = 0; i < mm; ++i) o.xy[i] = {x[i], y[i]};
    o.z.assign(z, z + zn);
    const UpdateReport r = static_cast<TerrainModel*>(m)->recursive_update(o, allow_birth != 0);
    rep[0] = r.active_blocks;
    rep[1] = r.active_centers;
    rep[2] = r.born_centers;
    rep[3] = r.rejected ? 1 : 0;
  });
}

int orc_fit_batch_ridge(const KP* k, const CP* c, const double* cx, const double* cy,
                        size_t n, const double* x, const double* y, const double* z,
                        size_t m, void** out) {
  return guarded([&] {
    *out = new TerrainModel(fit_batch_ridge(to_kp(k), to_cs(c, cx, cy, n), to_obs(x, y, z, m)));
  });
}

int orc_model_save(void* m, const char* path) {
  return guarded([&] { static_cast<TerrainModel*>(m)->save(path); });
}
int orc_model_load(const char* path, void** out) {
  return guarded([&] { *out = new TerrainModel(TerrainModel::load(path)); });
}

// ---- manifold rows + normal equations (contact.cpp, scan_matcher.cpp) ----------
// R row-major 3x3, t[3]; lever arms SoA hx/hy/hz. Outputs (nullable): r[n],
// J[6*n] (row i at J[6*i..]), valid[n], raw[n]; ne[29] = A upper-tri (21,
// row-major i<=j), g[6], cost, valid count.
int orc_manifold_rows(void* m, const double* R, const double* t, const double* hx,
                      const double* hy, const double* hz, size_t n, double wheel_radius,
                      double lambda_M, double huber, double* r, double* J,
                      unsigned char* valid, double* raw, double* ne29, int threads) {
  auto* tm = static_cast<TerrainModel*>(m);
  return guarded([&] {
    M3 RR;
    for (int i = 0; i < 9; ++i) RR.a[i] = R[i];
    const V3 tt{t[0], t[1], t[2]};
    std::vector<ManifoldRow> rows(n);
    auto work = [&](size_t b, size_t e) {
      for (size_t i = b; i < e; ++i)
        rows[i] = manifold_row(*tm, RR, tt, {hx[i], hy[i], hz[i]}, wheel_radius, lambda_M, huber);
    };
    if (threads <= 1) {
      work(0, n);
    } else {
      std::vector<std::thread> pool;
      const size_t chunk = (n + threads - 1) / threads;
      for (int w = 0; w < threads; ++w) {
        const size_t b = w * chunk, e = std::min(n, b + chunk);
        if (b < e) pool.emplace_back(work, b, e);
      }
      for (auto& th : pool) th.join();
    }
    NormalEq ne;
    for (size_t i = 0; i < n; ++i) {
      accumulate(ne, rows[i]);
      if (r) r[i] = rows[i].r;
      if (J)
        for (int c = 0; c < 6; ++c) J[6 * i + c] = rows[i].J[c];
      if (valid) valid[i] = rows[i].valid ? 1 : 0;
      if (raw) raw[i] = rows[i].raw;
    }
    if (ne29) {
      int k = 0;
      for (int i = 0; i < 6; ++i)
        for (int j = i; j < 6; ++j) ne29[k++] = ne.A[6 * i + j];
      for (int i = 0; i < 6; ++i) ne29[21 + i] = ne.g[i];
      ne29[27] = ne.cost;
      ne29[28] = static_cast<double>(ne.valid);
    }
  });
}

int orc_lm_step(const double* ne29, double mu, double* delta) {
  NormalEq ne;
  int k = 0;
  for (int i = 0; i < 6; ++i)
    for (int j = i; j < 6; ++j) {
      ne.A[6 * i + j] = ne29[k];
      ne.A[6 * j + i] = ne29[k];
      ++k;
    }
  for (int i = 0; i < 6; ++i) ne.g[i] = ne29[21 + i];
  return lm_step(ne, mu, delta) ? ORC_OK : ORC_RUNTIME_ERROR;
}

void orc_so3_exp(const double* w, double* R) {
  const M3 m = so3_exp({w[0], w[1], w[2]});
  std::memcpy(R, m.a, sizeof(m.a));
}

// pipeline.cpp:150-170 (out_* capacity >= max_points)
int orc_select_ground_points(const double* px, const double* py, const double* pz,
                             const unsigned char* kind, size_t n, const double* R,
                             const double* t, const double* roi, double radius, double voxel,
                             size_t max_points, double* ox, double* oy, double* oz,
                             size_t* out_n) {
  return guarded([&] {
    std::vector<V3> p(n);
    for (size_t i = 0; i < n; ++i) p[i] = {px[i], py[i], pz[i]};
    std::vector<std::uint8_t> k(kind, kind + n);
    M3 m;
    std::memcpy(m.a, R, sizeof(m.a));
    const Rect r{{roi[0], roi[1]}, {roi[2], roi[3]}};
    const GroundPoints g = select_ground_points(p, k, m, {t[0], t[1], t[2]}, r, radius, voxel,
                                                max_points);
    for (size_t i = 0; i < g.xy.size(); ++i) {
      ox[i] = g.xy[i].x;
      oy[i] = g.xy[i].y;
      oz[i] = g.z[i];
    }
    *out_n = g.xy.size();
  });
}

// metrics.cpp:199-232
int orc_terrain_error_histogram(void* m, const double* x, const double* y, const double* z,
                                size_t n, double trim, int bins, double* edges,
                                unsigned long long* counts, unsigned long long* trimmed,
                                unsigned long long* overflow) {
  auto* t = static_cast<TerrainModel*>(m);
  return guarded([&] {
    std::vector<V2> xy(n);
    for (size_t i = 0; i < n; ++i) xy[i] = {x[i], y[i]};
    const Histogram h = terrain_error_histogram(*t, xy, std::vector<double>(z, z + n), trim, bins);
    for (int b = 0; b <= bins; ++b) edges[b] = h.edges[b];
    for (int b = 0; b < bins; ++b) counts[b] = h.counts[b];
    *trimmed = h.trimmed;
    *overflow = h.overflow;
  });
}

// terrain_model.cpp:255-267 (numbers of export_csv); returns the point count
size_t orc_export_grid(void* m, double step, double* x, double* y, double* z, size_t cap) {
  auto* t = static_cast<TerrainModel*>(m);
  std::vector<double> xs, ys, zs;
  export_grid(*t, step, xs, ys, zs);
  for (size_t i = 0; i < xs.size() && i < cap; ++i) {
    x[i] = xs[i];
    y[i] = ys[i];
    z[i] = zs[i];
  }
  return xs.size();
}


// ---- feature correspondences (scan_matcher.cpp:44-216, local_map.cpp) ------
void* orc_map_new(double voxel, size_t window) {
  MapConfig c;
  c.voxel_size = voxel;
  c.window = window;
  return new LocalMap(c);
}
void orc_map_free(void* m) { delete static_cast<LocalMap*>(m); }
static FeatureInput to_features(const double* px, const double* py, const double* pz,
                                const unsigned char* kind, const int* label, size_t n) {
  FeatureInput f;
  f.p.resize(n);
  f.kind.assign(kind, kind + n);
  f.label.assign(n, -1);
  for (size_t i = 0; i < n; ++i) {
    f.p[i] = {px[i], py[i], pz[i]};
    if (label) f.label[i] = label[i];
  }
  return f;
}
static M3 to_m3(const double* R) {
  M3 m;
  std::memcpy(m.a, R, sizeof(m.a));
  return m;
}
void orc_map_insert(void* m, const double* px, const double* py, const double* pz,
                    const unsigned char* kind, const int* label, size_t n, const double* R,
                    const double* t) {
  static_cast<LocalMap*>(m)->insert(to_features(px, py, pz, kind, label, n), to_m3(R),
                                    {t[0], t[1], t[2]});
}
// kind 0 edge / 1 planar: count, and if xyz != NULL the points (cap) + labels
size_t orc_map_points(void* m, int kind, double* xyz, int* labels, size_t cap) {
  auto* mp = static_cast<LocalMap*>(m);
  const auto& pts = kind == 0 ? mp->edge : mp->planar;
  const auto& lab = kind == 0 ? mp->edge_label : mp->planar_label;
  for (size_t i = 0; xyz && i < pts.size() && i < cap; ++i) {
    xyz[3 * i] = pts[i].x;
    xyz[3 * i + 1] = pts[i].y;
    xyz[3 * i + 2] = pts[i].z;
    if (labels) labels[i] = lab[i];
  }
  return pts.size();
}
// tree: 1 = the kd-tree (reference algorithm), 0 = exhaustive cross-check
size_t orc_knn(void* m, int kind, double qx, double qy, double qz, int k, double gate,
               unsigned* out, int tree) {
  auto* mp = static_cast<LocalMap*>(m);
  const auto ids = tree ? (kind == 0 ? mp->edge_tree : mp->planar_tree).knn({qx, qy, qz}, k, gate)
                        : knn(kind == 0 ? mp->edge : mp->planar, {qx, qy, qz}, k, gate);
  for (size_t i = 0; i < ids.size(); ++i) out[i] = ids[i];
  return ids.size();
}
// cfg: corr_gate, huber_delta, plane_fit_tol, plane_eig_ratio, edge_eig_ratio,
// edge_fit_tol, edge_min_extent, trim_ratio, trim_floor, ground_corr_voxel,
// ground_corr_radius. Outputs (capacity n): kind, feature index, params[7]
// (edge: point xyz, dir xyz, 0; plane: normal xyz, offset, 0, 0, 0), weight,
// label, dist, fitq.
size_t orc_build_correspondences(void* m, const double* px, const double* py, const double* pz,
                                 const unsigned char* kind, size_t n, const double* R,
                                 const double* t, const double* cfg, int* ckind,
                                 unsigned* cfeat, double* params, double* weight, int* label,
                                 double* dist, double* fitq) {
  SolverConfigM c;
  c.corr_gate = cfg[0];
  c.huber_delta = cfg[1];
  c.plane_fit_tol = cfg[2];
  c.plane_eig_ratio = cfg[3];
  c.edge_eig_ratio = cfg[4];
  c.edge_fit_tol = cfg[5];
  c.edge_min_extent = cfg[6];
  c.trim_ratio = cfg[7];
  c.trim_floor = cfg[8];
  c.ground_corr_voxel = cfg[9];
  c.ground_corr_radius = cfg[10];
  const auto out = build_correspondences(to_features(px, py, pz, kind, nullptr, n), to_m3(R),
                                         {t[0], t[1], t[2]}, *static_cast<LocalMap*>(m), c);
  for (size_t i = 0; i < out.size(); ++i) {
    const auto& o = out[i];
    ckind[i] = o.kind;
    cfeat[i] = o.feature;
    double* pr = params + 7 * i;
    if (o.kind == 0) {
      pr[0] = o.line_point.x; pr[1] = o.line_point.y; pr[2] = o.line_point.z;
      pr[3] = o.line_dir.x; pr[4] = o.line_dir.y; pr[5] = o.line_dir.z; pr[6] = 0.0;
    } else {
      pr[0] = o.normal.x; pr[1] = o.normal.y; pr[2] = o.normal.z; pr[3] = o.offset;
      pr[4] = pr[5] = pr[6] = 0.0;
    }
    weight[i] = o.weight;
    label[i] = o.label;
    dist[i] = o.dist;
    fitq[i] = o.fitq;
  }
  return out.size();
}
// feature rows of total_cost at (R, t) -> ne29 (A upper 21, g 6, cost, rows)
void orc_feature_normal_eq(size_t nc, const int* ckind, const double* ps, const double* params,
                           const double* weight, const double* R, const double* t, double* ne29) {
  std::vector<Correspondence> cs(nc);
  for (size_t i = 0; i < nc; ++i) {
    auto& c = cs[i];
    c.kind = ckind[i];
    c.p_sensor = {ps[3 * i], ps[3 * i + 1], ps[3 * i + 2]};
    const double* pr = params + 7 * i;
    if (c.kind == 0) {
      c.line_point = {pr[0], pr[1], pr[2]};
      c.line_dir = {pr[3], pr[4], pr[5]};
    } else {
      c.normal = {pr[0], pr[1], pr[2]};
      c.offset = pr[3];
    }
    c.weight = weight[i];
  }
  NormalEq ne;
  size_t rows = 0;
  feature_normal_eq(cs, to_m3(R), {t[0], t[1], t[2]}, ne, &rows);
  int k = 0;
  for (int i = 0; i < 6; ++i)
    for (int j = i; j < 6; ++j) ne29[k++] = ne.A[6 * i + j];
  for (int i = 0; i < 6; ++i) ne29[21 + i] = ne.g[i];
  ne29[27] = ne.cost;
  ne29[28] = static_cast<double>(rows);
}

}  // extern "C"
