// TEST INFRASTRUCTURE — the same orc_* C entry points as oracle_capi.cpp,
// but backed by the REFERENCE ITSELF: this file is linked with the unchanged
// sources under /root/reference/proj/core (compiled by oracle/Makefile's
// `ref` target against the minimal Eigen subset in oracle/eigen_subset and the
// json/doctest stand-ins in oracle/shims) into oracle/_ref/libterralio_ref.so.
// oracle/oracle.py exposes it as oracle.reference(); tests use it to pin the
// plain-C++ restatement (oracle/terralio_oracle.cpp) and the GPU path to the
// reference's own outputs.
//
// Where the reference keeps something private this file reaches it only
// through public API:
//   * centers_near (terrain_model.cpp:62-66) = the reference's GridIndex2 over
//     model.centers() with cell min(cutoff, 1e6) (rebuild_indexes, :53-60);
//   * set_weights: a snapshot round trip through TerrainModel::save/load with
//     the weight section replaced (snapshot.cpp:7-14 layout);
//   * batched manifold rows: kin::manifold_residual/jacobian via
//     match::total_cost with two fixed-link legs whose chain end is the lever
//     arm (leg_model.cpp:10-21 then gives h exactly), so the Huber / lambda_M
//     weighting is the reference's own (scan_matcher.cpp:221-248);
//   * the LM step is lm_solve's inner damped solve (scan_matcher.cpp:296-305),
//     restated here in the same Eigen expressions.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <unistd.h>
#include <vector>
#include <chrono>
#include <deque>
#include <span>
#include <unordered_set>

#include "terralio/eval/metrics.hpp"
#include "terralio/grid_index.hpp"
#include "terralio/imu/preintegration.hpp"
#include "terralio/kinematics/contact.hpp"
#include "terralio/match/scan_matcher.hpp"
#include "terralio/parallel.hpp"
#include "terralio/pipeline.hpp"
#include "terralio/sim/simulator.hpp"
#include "terralio/so3.hpp"
#include "terralio/terrain/terrain_model.hpp"

using namespace terralio;
using terrain::CenterSet;
using terrain::KernelParams;
using terrain::TerrainModel;
using terrain::TerrainObservation;

namespace {
thread_local std::string g_err;

enum {
  ORC_OK = 0,
  ORC_INVALID_ARGUMENT = 1,
  ORC_DOMAIN_ERROR = 2,
  ORC_NO_SUPPORTED_CENTERS = 3,
  ORC_RUNTIME_ERROR = 4,
  ORC_BUFFER_TOO_SMALL = 7,
  ORC_UNSUPPORTED = 9,
};

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return ORC_OK;
  } catch (const terrain::NoSupportedCenters& e) {
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
  for (size_t i = 0; i < n; ++i) s.centers[i] = Vec2(cx[i], cy[i]);
  return s;
}
TerrainObservation to_obs(const double* x, const double* y, const double* z, size_t m, size_t zn) {
  TerrainObservation o;
  o.xy.resize(m);
  o.z.assign(z, z + zn);
  for (size_t i = 0; i < m; ++i) o.xy[i] = Vec2(x[i], y[i]);
  return o;
}
Mat3 to_m3(const double* R) {  // row-major
  Mat3 m;
  m << R[0], R[1], R[2], R[3], R[4], R[5], R[6], R[7], R[8];
  return m;
}

// A model plus the reference's own centre index (for centers_near).
struct RefModel {
  TerrainModel m;
  std::unique_ptr<GridIndex2> index;
  void reindex() {
    const double cell = std::min(m.kernel().cutoff_radius, 1e6);
    index = std::make_unique<GridIndex2>(cell);
    index->build(m.centers().centers);
  }
};
RefModel* wrap(TerrainModel&& t) {
  auto* r = new RefModel{std::move(t), nullptr};
  r->reindex();
  return r;
}
RefModel* M(void* h) { return static_cast<RefModel*>(h); }

std::string temp_path(const char* tag) {
  static std::atomic<unsigned> seq{0};
  const char* dir = std::getenv("TMPDIR");
  return std::string(dir ? dir : "/tmp") + "/tlg_ref_" + tag + "_" + std::to_string(::getpid()) + "_" +
         std::to_string(seq.fetch_add(1)) + ".bin";
}

// A leg whose chain end (base frame) is h: one fixed link with offset h.
kin::LegChain fixed_chain(double hx, double hy, double hz) {
  kin::LegChain c;
  kin::Link l;
  l.name = "wheel";
  l.offset = Vec3(hx, hy, hz);
  l.revolute = false;
  c.links.push_back(l);
  return c;
}

void pack_ne(const Eigen::MatrixXd& J, const Eigen::VectorXd& r, double cost, double rows, double* ne29) {
  const Eigen::Matrix<double, 6, 6> A = J.transpose() * J;
  const Eigen::Matrix<double, 6, 1> g = J.transpose() * r;
  int k = 0;
  for (int i = 0; i < 6; ++i)
    for (int j = i; j < 6; ++j) ne29[k++] = A(i, j);
  for (int i = 0; i < 6; ++i) ne29[21 + i] = g(i);
  ne29[27] = cost;
  ne29[28] = rows;
}

FeatureCloud to_cloud(const double* px, const double* py, const double* pz, const unsigned char* kind,
                      const int* label, size_t n) {
  FeatureCloud f;
  f.points.resize(n);
  for (size_t i = 0; i < n; ++i) {
    f.points[i].p = Vec3(px[i], py[i], pz[i]);
    f.points[i].kind = static_cast<FeatureKind>(kind[i]);
    f.points[i].label = label ? label[i] : -1;
  }
  return f;
}

match::SolverConfig to_solver(const double* cfg) {
  match::SolverConfig c;
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
  return c;
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
const char* orc_backend() { return "reference"; }

// ---- RNG: std::mt19937_64 with libstdc++ distributions (as the port) -------
void* orc_rng_new(unsigned long long seed) { return new std::mt19937_64(seed); }
void orc_rng_free(void* r) { delete static_cast<std::mt19937_64*>(r); }
void orc_uniform(void* r, double lo, double hi, size_t n, double* out) {
  std::uniform_real_distribution<double> d(lo, hi);
  auto& g = *static_cast<std::mt19937_64*>(r);
  for (size_t i = 0; i < n; ++i) out[i] = d(g);
}
int orc_uniform_int(void* r, int lo, int hi) {
  std::uniform_int_distribution<int> d(lo, hi);
  return d(*static_cast<std::mt19937_64*>(r));
}
void* orc_normal_new(double mean, double sd) { return new std::normal_distribution<double>(mean, sd); }
void orc_normal_free(void* d) { delete static_cast<std::normal_distribution<double>*>(d); }
void orc_normal(void* d, void* r, size_t n, double* out) {
  auto& nd = *static_cast<std::normal_distribution<double>*>(d);
  auto& g = *static_cast<std::mt19937_64*>(r);
  for (size_t i = 0; i < n; ++i) out[i] = nd(g);
}

// ---- kernel.cpp ----------------------------------------------------------------
int orc_kernel_finalize(KP* k) {
  return guarded([&] {
    KernelParams p = to_kp(k);
    p.finalize();
    k->cutoff_radius = p.cutoff_radius;
  });
}
int orc_kernel_eval(const KP* k, double xx, double xy, double cx, double cy, double bw, double* out) {
  return guarded([&] { *out = terrain::kernel_eval(to_kp(k), Vec2(xx, xy), Vec2(cx, cy), bw); });
}
double orc_sigma_tilde(const KP* k) { return to_kp(k).sigma_tilde(); }
double orc_moment_scale(const KP* k) { return to_kp(k).moment_scale(); }

// ---- grid_index.hpp --------------------------------------------------------------
void* orc_grid_new(double cell, const double* x, const double* y, size_t n) {
  auto* g = new GridIndex2(cell);
  for (size_t i = 0; i < n; ++i) g->insert(Vec2(x[i], y[i]));
  return g;
}
void orc_grid_free(void* g) { delete static_cast<GridIndex2*>(g); }
size_t orc_grid_query(void* g, double qx, double qy, double r, unsigned* out, size_t cap) {
  const auto ids = static_cast<GridIndex2*>(g)->radius_query(Vec2(qx, qy), r);
  for (size_t i = 0; i < ids.size() && i < cap; ++i) out[i] = ids[i];
  return ids.size();
}

// ---- center_select.cpp -----------------------------------------------------------
int orc_supported_mesh_nodes(const double* x, const double* y, const double* z, size_t m, size_t zn,
                             double rminx, double rminy, double rmaxx, double rmaxy, double res,
                             double r_a, int count, int throw_empty, double* out_x, double* out_y,
                             size_t cap, size_t* out_n) {
  return guarded([&] {
    const TerrainObservation o = to_obs(x, y, z, m, zn);
    const Rect roi{Vec2(rminx, rminy), Vec2(rmaxx, rmaxy)};
    const std::vector<Vec2> nodes = throw_empty ? terrain::select_centers(o, roi, res, r_a, count).centers
                                                : terrain::supported_mesh_nodes(o, roi, res, r_a, count);
    *out_n = nodes.size();
    if (nodes.size() > cap) throw std::length_error("buffer too small");
    for (size_t i = 0; i < nodes.size(); ++i) {
      out_x[i] = nodes[i].x();
      out_y[i] = nodes[i].y();
    }
  });
}

// ---- TerrainModel ------------------------------------------------------------------
int orc_model_new(const KP* k, const CP* c, const double* cx, const double* cy, size_t n, void** out) {
  return guarded([&] { *out = wrap(TerrainModel(to_kp(k), to_cs(c, cx, cy, n))); });
}
void orc_model_free(void* m) { delete M(m); }
size_t orc_model_num_centers(void* m) { return M(m)->m.num_centers(); }
size_t orc_model_num_blocks(void* m) { return M(m)->m.num_blocks(); }
void orc_model_kernel(void* m, KP* k) {
  const auto& p = M(m)->m.kernel();
  *k = {p.sigma, p.sigma_eps, p.lambda, p.cutoff_radius};
}
void orc_model_centers(void* m, double* cx, double* cy) {
  const auto& c = M(m)->m.centers().centers;
  for (size_t i = 0; i < c.size(); ++i) {
    cx[i] = c[i].x();
    cy[i] = c[i].y();
  }
}
void orc_model_weights(void* m, double* w) {
  const auto& v = M(m)->m.weights();
  for (Eigen::Index i = 0; i < v.size(); ++i) w[i] = v(i);
}
// snapshot round trip with the weight section replaced (snapshot.cpp:7-14:
// 16-byte header, N centre pairs, then N weights)
int orc_model_set_weights(void* m, const double* w) {
  return guarded([&] {
    RefModel* r = M(m);
    const std::string path = temp_path("w");
    r->m.save(path);
    const size_t n = r->m.num_centers();
    {
      std::fstream f(path, std::ios::in | std::ios::out | std::ios::binary);
      f.seekp(16 + static_cast<std::streamoff>(16 * n));
      f.write(reinterpret_cast<const char*>(w), static_cast<std::streamsize>(8 * n));
    }
    r->m = TerrainModel::load(path);
    std::remove(path.c_str());
    r->reindex();
  });
}
// replace block b's info_inv (column-major bn x bn; its lower triangle is
// what the snapshot stores, row-major, snapshot.cpp:13) by a round trip
int orc_model_set_block_info_inverse(void* m, unsigned b, const double* a) {
  return guarded([&] {
    RefModel* r = M(m);
    const size_t n = r->m.num_centers();
    if (b >= r->m.num_blocks()) throw std::invalid_argument("block id out of range");
    std::streamoff off = 16 + static_cast<std::streamoff>(28 * n);
    for (unsigned q = 0; q < b; ++q) {
      const auto bn = static_cast<std::streamoff>(r->m.block_members(q).size());
      off += 8 * bn * (bn + 1) / 2;
    }
    const size_t bn = r->m.block_members(b).size();
    std::vector<double> tri;
    for (size_t i = 0; i < bn; ++i)
      for (size_t j = 0; j <= i; ++j) tri.push_back(a[i + j * bn]);
    const std::string path = temp_path("ii");
    r->m.save(path);
    {
      std::fstream f(path, std::ios::in | std::ios::out | std::ios::binary);
      f.seekp(off);
      f.write(reinterpret_cast<const char*>(tri.data()), static_cast<std::streamsize>(8 * tri.size()));
    }
    r->m = TerrainModel::load(path);
    std::remove(path.c_str());
    r->reindex();
  });
}
void orc_model_block_index(void* m, unsigned* out) {
  const TerrainModel& t = M(m)->m;
  for (size_t i = 0; i < t.num_centers(); ++i) out[i] = t.block_of(static_cast<unsigned>(i));
}
size_t orc_model_block_size(void* m, unsigned b) { return M(m)->m.block_members(b).size(); }
void orc_model_block_members(void* m, unsigned b, unsigned* out) {
  const auto& v = M(m)->m.block_members(b);
  for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
}
void orc_model_block_info_inverse(void* m, unsigned b, double* out) {  // column-major
  const Eigen::MatrixXd& a = M(m)->m.block_info_inverse(b);
  for (Eigen::Index j = 0; j < a.cols(); ++j)
    for (Eigen::Index i = 0; i < a.rows(); ++i) out[i + j * a.rows()] = a(i, j);
}

int orc_model_predict(void* m, const double* x, const double* y, size_t n, double* z, unsigned char* sup,
                      double* gx, double* gy, int threads) {
  const TerrainModel& t = M(m)->m;
  return guarded([&] {
    auto work = [&](size_t b, size_t e) {
      for (size_t i = b; i < e; ++i) {
        if (z || sup) {
          const terrain::HeightQuery q = t.predict_height(Vec2(x[i], y[i]));
          if (z) z[i] = q.z;
          if (sup) sup[i] = q.supported ? 1 : 0;
        }
        if (gx || gy) {
          const Vec2 g = t.predict_gradient(Vec2(x[i], y[i]));
          if (gx) gx[i] = g.x();
          if (gy) gy[i] = g.y();
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

// Parity scales, from the reference's neighbour index and
// weights: s = sum |w kappa_sigma|, g = sum |w kappa_sigma| d / sigma^2.
int orc_model_scales(void* m, const double* x, const double* y, size_t n, double* s, double* g,
                     int threads) {
  RefModel* r = M(m);
  return guarded([&] {
    const double sig = r->m.kernel().sigma, cut = r->m.kernel().cutoff_radius;
    const Eigen::VectorXd& w = r->m.weights();
    const auto& c = r->m.centers().centers;
    auto work = [&](size_t b, size_t e) {
      for (size_t i = b; i < e; ++i) {
        double a = 0.0, q = 0.0;
        for (std::uint32_t id : r->index->radius_query(Vec2(x[i], y[i]), cut)) {
          const double dx = x[i] - c[id].x(), dy = y[i] - c[id].y();
          const double d2 = dx * dx + dy * dy;
          const double v = std::abs(w(id) * std::exp(-d2 / (2.0 * sig * sig)));
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
  RefModel* r = M(m);
  const auto ids = r->index->radius_query(Vec2(qx, qy), r->m.kernel().cutoff_radius);
  for (size_t i = 0; i < ids.size() && i < cap; ++i) out[i] = ids[i];
  return ids.size();
}

int orc_model_moment_feature(void* m, double qx, double qy, unsigned* ids, double* vals, size_t cap,
                             size_t* out_n) {
  return guarded([&] {
    const terrain::SparseVec f = M(m)->m.moment_feature(Vec2(qx, qy));
    *out_n = f.entries.size();
    for (size_t i = 0; i < f.entries.size() && i < cap; ++i) {
      ids[i] = f.entries[i].first;
      vals[i] = f.entries[i].second;
    }
  });
}

int orc_model_recursive_update(void* m, const double* x, const double* y, const double* z, size_t mm,
                               size_t zn, int allow_birth, unsigned long long* rep) {
  return guarded([&] {
    RefModel* r = M(m);
    const terrain::UpdateReport u = r->m.recursive_update(to_obs(x, y, z, mm, zn), allow_birth != 0);
    if (u.born_centers) r->reindex();
    rep[0] = u.active_blocks;
    rep[1] = u.active_centers;
    rep[2] = u.born_centers;
    rep[3] = u.rejected ? 1 : 0;
  });
}

int orc_fit_batch_ridge(const KP* k, const CP* c, const double* cx, const double* cy, size_t n,
                        const double* x, const double* y, const double* z, size_t m, void** out) {
  return guarded([&] {
    *out = wrap(terrain::fit_batch_ridge(to_kp(k), to_cs(c, cx, cy, n), to_obs(x, y, z, m, m)));
  });
}

int orc_model_save(void* m, const char* path) {
  return guarded([&] { M(m)->m.save(path); });
}
int orc_model_load(const char* path, void** out) {
  return guarded([&] { *out = wrap(TerrainModel::load(path)); });
}
int orc_model_export_csv(void* m, const char* path, double step) {
  return guarded([&] { M(m)->m.export_csv(path, step); });
}

// ---- manifold rows + normal equations -------------------------------------------
// Lever arms are taken two at a time as the (left, right) wheels of one
// match::total_cost evaluation with no correspondences.
int orc_manifold_rows(void* m, const double* R, const double* t, const double* hx, const double* hy,
                      const double* hz, size_t n, double wheel_radius, double lambda_M, double huber,
                      double* r, double* J, unsigned char* valid, double* raw, double* ne29, int threads) {
  const TerrainModel& tm = M(m)->m;
  return guarded([&] {
    RobotState state;
    state.rotation = to_m3(R);
    state.translation = Vec3(t[0], t[1], t[2]);
    match::SolverConfig cfg;
    cfg.lambda_manifold = lambda_M;
    cfg.manifold_huber_delta = huber;
    Eigen::MatrixXd Jall = Eigen::MatrixXd::Zero(static_cast<Eigen::Index>(n), 6);
    Eigen::VectorXd rall = Eigen::VectorXd::Zero(static_cast<Eigen::Index>(n));
    std::vector<unsigned char> vall(n, 0);
    std::vector<double> rawall(n, 0.0);
    auto work = [&](size_t b, size_t e) {
      JointConfig joints;
      for (size_t i = b; i < e; i += 2) {
        const size_t j = (i + 1 < e) ? i + 1 : i;
        kin::LegModel leg;
        leg.wheel_radius = wheel_radius;
        leg.left = fixed_chain(hx[i], hy[i], hz[i]);
        leg.right = fixed_chain(hx[j], hy[j], hz[j]);
        match::ManifoldInputs mi{&joints, &leg, &tm};
        match::CostEval ev;
        try {
          ev = match::total_cost(state, {}, mi, cfg);
        } catch (const std::runtime_error&) {
          continue;  // both rows unsupported: "nothing to optimize", zero rows
        }
        const size_t ids[2] = {i, j};
        const std::optional<double> raws[2] = {ev.manifold_left, ev.manifold_right};
        for (int s = 0; s < (j == i ? 1 : 2); ++s) {
          const size_t k = ids[s];
          rall(static_cast<Eigen::Index>(k)) = ev.residual(s);
          for (int c = 0; c < 6; ++c) Jall(static_cast<Eigen::Index>(k), c) = ev.jacobian(s, c);
          vall[k] = raws[s].has_value() ? 1 : 0;
          rawall[k] = raws[s].value_or(0.0);
        }
      }
    };
    // pairs never straddle two workers (even chunk sizes)
    if (threads <= 1) {
      work(0, n);
    } else {
      std::vector<std::thread> pool;
      size_t chunk = (n + threads - 1) / threads;
      chunk += chunk & 1;
      for (int w = 0; w < threads; ++w) {
        const size_t b = w * chunk, e = std::min(n, b + chunk);
        if (b < e) pool.emplace_back(work, b, e);
      }
      for (auto& th : pool) th.join();
    }
    size_t nvalid = 0;
    for (size_t i = 0; i < n; ++i) {
      nvalid += vall[i];
      if (r) r[i] = rall(static_cast<Eigen::Index>(i));
      if (J)
        for (int c = 0; c < 6; ++c) J[6 * i + c] = Jall(static_cast<Eigen::Index>(i), c);
      if (valid) valid[i] = vall[i];
      if (raw) raw[i] = rawall[i];
    }
    if (ne29) pack_ne(Jall, rall, rall.squaredNorm(), static_cast<double>(nvalid), ne29);
  });
}

// lm_solve's damped step (scan_matcher.cpp:296-305)
int orc_lm_step(const double* ne29, double mu, double* delta_out) {
  Eigen::Matrix<double, 6, 6> A;
  int k = 0;
  for (int i = 0; i < 6; ++i)
    for (int j = i; j < 6; ++j) {
      A(i, j) = ne29[k];
      A(j, i) = ne29[k];
      ++k;
    }
  Eigen::Matrix<double, 6, 1> g;
  for (int i = 0; i < 6; ++i) g(i) = ne29[21 + i];
  Eigen::Matrix<double, 6, 6> damped = A;
  damped.diagonal() += mu * A.diagonal().cwiseMax(1e-12);
  damped.diagonal().array() += 1e-3;
  const Eigen::Matrix<double, 6, 1> delta = -damped.ldlt().solve(g);
  for (int i = 0; i < 6; ++i) delta_out[i] = delta(i);
  return delta.allFinite() ? ORC_OK : ORC_RUNTIME_ERROR;
}

void orc_so3_exp(const double* w, double* R) {
  const Mat3 m = so3_exp(Vec3(w[0], w[1], w[2]));
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R[3 * i + j] = m(i, j);
}

// pipeline.cpp's select_ground_points is file-local in the reference.
int orc_select_ground_points(const double*, const double*, const double*, const unsigned char*, size_t,
                             const double*, const double*, const double*, double, double, size_t,
                             double*, double*, double*, size_t*) {
  g_err = "select_ground_points is file-local in the reference (pipeline.cpp:150)";
  return ORC_UNSUPPORTED;
}

// metrics.cpp:199-232
int orc_terrain_error_histogram(void* m, const double* x, const double* y, const double* z, size_t n,
                                double trim, int bins, double* edges, unsigned long long* counts,
                                unsigned long long* trimmed, unsigned long long* overflow) {
  return guarded([&] {
    std::vector<Vec2> xy(n);
    for (size_t i = 0; i < n; ++i) xy[i] = Vec2(x[i], y[i]);
    const eval::Histogram h =
        eval::terrain_error_histogram(M(m)->m, xy, std::vector<double>(z, z + n), trim, bins);
    for (int b = 0; b <= bins; ++b) edges[b] = h.edges[static_cast<size_t>(b)];
    for (int b = 0; b < bins; ++b) counts[b] = h.counts[static_cast<size_t>(b)];
    *trimmed = h.trimmed;
    *overflow = h.overflow;
  });
}

// export_csv's grid walk (terrain_model.cpp:255-267) parsed back from the file
size_t orc_export_grid(void* m, double step, double* x, double* y, double* z, size_t cap) {
  const std::string path = temp_path("csv");
  M(m)->m.export_csv(path, step);
  std::ifstream in(path);
  std::string line;
  std::getline(in, line);
  size_t k = 0;
  while (std::getline(in, line)) {
    double a, b, c;
    if (std::sscanf(line.c_str(), "%lf,%lf,%lf", &a, &b, &c) != 3) continue;
    if (k < cap) {
      x[k] = a;
      y[k] = b;
      z[k] = c;
    }
    ++k;
  }
  std::remove(path.c_str());
  return k;
}

// ---- feature correspondences (scan_matcher.cpp:44-216, local_map.cpp) --------
void* orc_map_new(double voxel, size_t window) {
  match::MapConfig c;
  c.voxel_size = voxel;
  c.window = window;
  return new match::LocalMap(c);
}
void orc_map_free(void* m) { delete static_cast<match::LocalMap*>(m); }
void orc_map_insert(void* m, const double* px, const double* py, const double* pz, const unsigned char* kind,
                    const int* label, size_t n, const double* R, const double* t) {
  static_cast<match::LocalMap*>(m)->insert(to_cloud(px, py, pz, kind, label, n), to_m3(R),
                                           Vec3(t[0], t[1], t[2]));
}
size_t orc_map_points(void* m, int kind, double* xyz, int* labels, size_t cap) {
  auto* mp = static_cast<match::LocalMap*>(m);
  const KdTree3& tree = kind == 0 ? mp->edge_tree() : mp->planar_tree();
  for (size_t i = 0; xyz && i < tree.size() && i < cap; ++i) {
    const Vec3& p = tree.point(static_cast<std::uint32_t>(i));
    xyz[3 * i] = p.x();
    xyz[3 * i + 1] = p.y();
    xyz[3 * i + 2] = p.z();
    if (labels)
      labels[i] = kind == 0 ? mp->edge_label(static_cast<std::uint32_t>(i))
                            : mp->planar_label(static_cast<std::uint32_t>(i));
  }
  return tree.size();
}
size_t orc_knn(void* m, int kind, double qx, double qy, double qz, int k, double gate, unsigned* out,
               int /*tree*/) {
  auto* mp = static_cast<match::LocalMap*>(m);
  const auto ids = (kind == 0 ? mp->edge_tree() : mp->planar_tree()).knn(Vec3(qx, qy, qz), k, gate);
  for (size_t i = 0; i < ids.size(); ++i) out[i] = ids[i];
  return ids.size();
}
// Outputs as the port; the feature index is recovered from the scan order
// (build_correspondences emits in feature order), dist recomputed with the
// reference's residuals at the guess pose, fitq is not exposed (NaN).
size_t orc_build_correspondences(void* m, const double* px, const double* py, const double* pz,
                                 const unsigned char* kind, size_t n, const double* R, const double* t,
                                 const double* cfg, int* ckind, unsigned* cfeat, double* params,
                                 double* weight, int* label, double* dist, double* fitq) {
  const FeatureCloud f = to_cloud(px, py, pz, kind, nullptr, n);
  RobotState guess;
  guess.rotation = to_m3(R);
  guess.translation = Vec3(t[0], t[1], t[2]);
  const auto out = match::build_correspondences(f, guess, *static_cast<match::LocalMap*>(m), to_solver(cfg));
  size_t j = 0;
  for (size_t i = 0; i < out.size(); ++i) {
    const auto& o = out[i];
    while (j < n && !(f.points[j].p.x() == o.p_sensor.x() && f.points[j].p.y() == o.p_sensor.y() &&
                      f.points[j].p.z() == o.p_sensor.z() &&
                      ((o.kind == FeatureKind::Edge) == (f.points[j].kind == FeatureKind::Edge))))
      ++j;
    cfeat[i] = static_cast<unsigned>(j);
    ++j;
    ckind[i] = o.kind == FeatureKind::Edge ? 0 : 1;
    double* pr = params + 7 * i;
    const Vec3 pw = guess.rotation * o.p_sensor + guess.translation;
    if (o.kind == FeatureKind::Edge) {
      pr[0] = o.line.point.x();
      pr[1] = o.line.point.y();
      pr[2] = o.line.point.z();
      pr[3] = o.line.direction.x();
      pr[4] = o.line.direction.y();
      pr[5] = o.line.direction.z();
      pr[6] = 0.0;
      dist[i] = match::point_to_line_residual(pw, o.line).value.norm();
    } else {
      pr[0] = o.plane.normal.x();
      pr[1] = o.plane.normal.y();
      pr[2] = o.plane.normal.z();
      pr[3] = o.plane.offset;
      pr[4] = pr[5] = pr[6] = 0.0;
      dist[i] = std::abs(match::point_to_plane_residual(pw, o.plane).value);
    }
    weight[i] = o.weight;
    label[i] = o.map_label;
    fitq[i] = std::nan("");
  }
  return out.size();
}
// feature rows of total_cost at (R, t) -> ne29 (A upper 21, g 6, cost, rows)
void orc_feature_normal_eq(size_t nc, const int* ckind, const double* ps, const double* params,
                           const double* weight, const double* R, const double* t, double* ne29) {
  std::vector<match::Correspondence> cs(nc);
  for (size_t i = 0; i < nc; ++i) {
    auto& c = cs[i];
    c.kind = ckind[i] == 0 ? FeatureKind::Edge : FeatureKind::Planar;
    c.p_sensor = Vec3(ps[3 * i], ps[3 * i + 1], ps[3 * i + 2]);
    const double* pr = params + 7 * i;
    if (ckind[i] == 0) {
      c.line.point = Vec3(pr[0], pr[1], pr[2]);
      c.line.direction = Vec3(pr[3], pr[4], pr[5]);
    } else {
      c.plane.normal = Vec3(pr[0], pr[1], pr[2]);
      c.plane.offset = pr[3];
    }
    c.weight = weight[i];
  }
  RobotState s;
  s.rotation = to_m3(R);
  s.translation = Vec3(t[0], t[1], t[2]);
  std::memset(ne29, 0, 29 * sizeof(double));
  try {
    const match::CostEval ev = match::total_cost(s, cs, {}, match::SolverConfig{});
    pack_ne(ev.jacobian, ev.residual, ev.cost, static_cast<double>(ev.feature_rows), ne29);
  } catch (const std::runtime_error&) {
  }
}

// ---- reference simulator bundles, lm_solve and the odometry loop --------------
// (pose-level parity: scan_matcher.cpp:257-358, pipeline.cpp:196-300)

// sim::simulate on a stock scene (scene.cpp:151-168) with an optional
// ScanConfig override (azimuth x elevation rays), kept to the first scans.
void* ref_sim_new(const char* scene, unsigned long long seed, int az, int el, long max_scans) {
  try {
    sim::Scene sc = sim::stock_scene(scene);
    if (az > 0) sc.scan.azimuth_steps = az;
    if (el > 0) sc.scan.elevation_steps = el;
    auto* b = new sim::SequenceBundle(sim::simulate(sc, seed));
    if (max_scans > 0 && b->scans.size() > static_cast<size_t>(max_scans)) {
      b->scans.resize(static_cast<size_t>(max_scans));
      b->gt_poses.resize(static_cast<size_t>(max_scans));
    }
    return b;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void ref_sim_free(void* b) { delete static_cast<sim::SequenceBundle*>(b); }
size_t ref_sim_num_scans(void* b) { return static_cast<sim::SequenceBundle*>(b)->scans.size(); }
// returns the point count; fills up to cap
size_t ref_sim_scan(void* b, size_t k, double* px, double* py, double* pz, unsigned char* kind, int* label,
                    size_t cap) {
  const auto& pts = static_cast<sim::SequenceBundle*>(b)->scans[k].points;
  for (size_t i = 0; i < pts.size() && i < cap; ++i) {
    px[i] = pts[i].p.x();
    py[i] = pts[i].p.y();
    pz[i] = pts[i].p.z();
    kind[i] = static_cast<unsigned char>(pts[i].kind);
    label[i] = pts[i].label;
  }
  return pts.size();
}
void ref_sim_gt(void* b, size_t k, double* R9, double* t3, double* ts) {
  const TimedPose& p = static_cast<sim::SequenceBundle*>(b)->gt_poses[k];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R9[3 * i + j] = p.rotation(i, j);
  for (int i = 0; i < 3; ++i) t3[i] = p.translation(i);
  *ts = p.timestamp;
}
void ref_sim_roi(void* b, double* roi4) {
  const Rect& r = static_cast<sim::SequenceBundle*>(b)->scene.terrain_roi;
  roi4[0] = r.min.x();
  roi4[1] = r.min.y();
  roi4[2] = r.max.x();
  roi4[3] = r.max.y();
}
double ref_sim_wheel_radius(void* b) { return static_cast<sim::SequenceBundle*>(b)->robot.wheel_radius; }

namespace {
// pipeline.cpp:176-186 (file-local there)
const JointConfig* nearest_joints_(const std::vector<JointConfig>& joints, double t) {
  if (joints.empty()) return nullptr;
  const auto it = std::lower_bound(joints.begin(), joints.end(), t,
                                   [](const JointConfig& j, double v) { return j.timestamp < v; });
  if (it == joints.begin()) return &*it;
  if (it == joints.end()) return &joints.back();
  return (it->timestamp - t < t - std::prev(it)->timestamp) ? &*it : &*std::prev(it);
}
// pipeline.cpp:164-174
std::span<const ImuSample> imu_window_(const std::vector<ImuSample>& imu, double t0, double t1) {
  const auto begin = std::lower_bound(imu.begin(), imu.end(), t0,
                                      [](const ImuSample& s, double t) { return s.timestamp <= t; });
  const auto end = std::upper_bound(begin, imu.end(), t1,
                                    [](double t, const ImuSample& s) { return t < s.timestamp - 1e-9; });
  return {&*begin, static_cast<std::size_t>(end - begin)};
}
// pipeline.cpp:150-170
terrain::TerrainObservation select_ground_points_(const FeatureCloud& scan, const Mat3& R, const Vec3& t,
                                                  const Rect& roi, const pipeline::RunConfig& cfg) {
  terrain::TerrainObservation obs;
  std::unordered_set<std::int64_t> voxels;
  for (const FeaturePoint& f : scan.points) {
    if (f.kind != FeatureKind::Ground) continue;
    const Vec3 p = R * f.p + t;
    const Vec2 xy = p.head<2>();
    if (!roi.contains(xy)) continue;
    if ((xy - t.head<2>()).norm() > cfg.ground_radius) continue;
    const auto vx = static_cast<std::int64_t>(std::floor(xy.x() / cfg.ground_voxel));
    const auto vy = static_cast<std::int64_t>(std::floor(xy.y() / cfg.ground_voxel));
    if (!voxels.insert((vx << 21) ^ (vy & ((1 << 21) - 1))).second) continue;
    obs.xy.push_back(xy);
    obs.z.push_back(p.z());
    if (obs.xy.size() >= cfg.ground_max_points) break;
  }
  return obs;
}
void put_pose(double* out, const Mat3& R, const Vec3& t) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) out[3 * i + j] = R(i, j);
  for (int i = 0; i < 3; ++i) out[9 + i] = t(i);
}
}  // namespace

// Wheel-centre lever arms (base frame, leg_model.cpp:10-21) from the joint
// sample nearest t (pipeline.cpp:176-186); returns 0 when there is none.
int ref_sim_wheel_arms(void* bp, double t, double* hL, double* hR) {
  auto* b = static_cast<sim::SequenceBundle*>(bp);
  const JointConfig* j = nearest_joints_(b->joints, t);
  if (!j) return 0;
  for (const kin::Side side : {kin::Side::Left, kin::Side::Right}) {
    const kin::LegChain& chain = b->robot.chain(side);
    const int off = b->robot.joint_offset(side);
    const std::span<const double> q(j->angles.data() + off, static_cast<std::size_t>(chain.joint_count()));
    const Vec3 h = kin::chain_end_position(chain, q);
    double* o = side == kin::Side::Left ? hL : hR;
    for (int i = 0; i < 3; ++i) o[i] = h(i);
  }
  return 1;
}

// The odometry loop of pipeline.cpp:196-300 with per-frame records, in one
// of two modes: mode 1 calls pipeline::run_odometry itself (poses, wall ms
// and the solve/terrain reports come from its RunResult); mode 0 runs the
// same loop restated here from the reference's public pieces, additionally
// recording the predicted pose and the lever arms each lm_solve saw (what a
// lock-step comparison needs). `config_json` is RunConfig::from_json text.
// Per frame k: poses[12k] = (R row-major, t) solved, preds[12k] predicted,
// arms[7k] = hL, hR, has_joints; ints[8k] = held, inserted, converged,
// failed, degenerate, outer_iterations, accepted_steps, correspondences;
// terr[4k] = active_blocks, active_centers, born_centers, rejected;
// dbl[3k] = final_cost, wall_ms, smallest_feature_eigenvalue.
int ref_odometry(void* bp, const char* config_json, int mode, double* poses, double* preds, double* arms,
                 int* ints, double* terr, double* dbl) {
  return guarded([&] {
    const auto& bundle = *static_cast<sim::SequenceBundle*>(bp);
    const pipeline::RunConfig config = pipeline::RunConfig::from_json(config_json);
    const size_t nscan = bundle.scans.size();
    auto record = [&](size_t k, const pipeline::FrameDiagnostics& d, const Mat3& R, const Vec3& t) {
      put_pose(poses + 12 * k, R, t);
      int* o = ints + 8 * k;
      o[0] = d.held;
      o[1] = d.inserted;
      o[2] = d.solve.converged;
      o[3] = d.solve.failed;
      o[4] = d.solve.degenerate;
      o[5] = d.solve.outer_iterations;
      o[6] = d.solve.accepted_steps;
      o[7] = static_cast<int>(d.solve.correspondence_count);
      terr[4 * k] = static_cast<double>(d.terrain.active_blocks);
      terr[4 * k + 1] = static_cast<double>(d.terrain.active_centers);
      terr[4 * k + 2] = static_cast<double>(d.terrain.born_centers);
      terr[4 * k + 3] = d.terrain.rejected;
      dbl[3 * k] = d.solve.final_cost;
      dbl[3 * k + 1] = d.wall_ms;
      dbl[3 * k + 2] = d.solve.smallest_feature_eigenvalue;
    };
    if (mode == 1) {
      const pipeline::RunResult res = pipeline::run_odometry(bundle, config);
      for (size_t k = 0; k < nscan; ++k)
        record(k, res.frames[k], res.trajectory[k].rotation, res.trajectory[k].translation);
      return;
    }
    set_worker_count(static_cast<std::size_t>(config.workers));
    terrain::KernelParams kernel = config.kernel;
    kernel.finalize();
    terrain::CenterSet centers;
    centers.mesh_resolution = config.mesh_resolution;
    centers.accept_radius = config.accept_radius;
    centers.accept_count = config.accept_count;
    centers.roi = bundle.scene.terrain_roi;
    terrain::TerrainModel model(kernel, centers);
    match::LocalMap map(config.map);
    RobotState state;
    state.rotation = bundle.gt_poses.front().rotation;
    state.translation = bundle.gt_poses.front().translation;
    state.accel_bias = config.imu_biases.accel;
    state.gyro_bias = config.imu_biases.gyro;
    std::deque<double> cost_history;
    for (size_t k = 0; k < nscan; ++k) {
      const auto t_start = std::chrono::steady_clock::now();
      const FeatureCloud& scan = bundle.scans[k];
      const double t_k = bundle.gt_poses[k].timestamp;
      pipeline::FrameDiagnostics diag;
      diag.index = k;
      diag.timestamp = t_k;
      RobotState pred = state;
      double* ar = arms + 7 * k;
      std::fill(ar, ar + 7, 0.0);
      if (k > 0) {
        const double t_prev = bundle.gt_poses[k - 1].timestamp;
        const double dt = t_k - t_prev;
        if (config.use_imu) {
          const auto window = imu_window_(bundle.imu, t_prev, t_k);
          const auto delta = imu::preintegrate(window, t_prev, t_k, {state.accel_bias, state.gyro_bias});
          pred = imu::predict_pose(state, delta);
        } else {
          pred.translation += state.velocity * dt;
        }
        match::ManifoldInputs manifold;
        const JointConfig* joints = nearest_joints_(bundle.joints, t_k);
        if (config.use_manifold && joints) {
          manifold.joints = joints;
          manifold.leg = &bundle.robot;
          manifold.terrain = &model;
          ref_sim_wheel_arms(bp, t_k, ar, ar + 3);
          ar[6] = 1.0;
        }
        RobotState solved = match::lm_solve(pred, scan, map, manifold, config.solver, &diag.solve);
        if (diag.solve.failed) {
          solved = pred;
          diag.held = true;
        }
        solved.velocity = (solved.translation - state.translation) / dt;
        solved.accel_bias = state.accel_bias;
        solved.gyro_bias = state.gyro_bias;
        state = solved;
      }
      put_pose(preds + 12 * k, pred.rotation, pred.translation);
      bool accept = !diag.held;
      if (k > 0 && accept) {
        const double rows = std::max<std::size_t>(diag.solve.correspondence_count, 1);
        const double per_row = diag.solve.final_cost / rows;
        if (cost_history.size() >= 5) {
          std::vector<double> sorted(cost_history.begin(), cost_history.end());
          std::nth_element(sorted.begin(), sorted.begin() + sorted.size() / 2, sorted.end());
          const double med = sorted[sorted.size() / 2];
          if (per_row > std::max(10.0 * med, 1e-6)) accept = false;
        }
        if (accept) {
          cost_history.push_back(per_row);
          if (cost_history.size() > 20) cost_history.pop_front();
        }
      }
      diag.inserted = accept;
      if (accept) {
        map.insert(scan, state.rotation, state.translation);
        const auto obs = select_ground_points_(scan, state.rotation, state.translation,
                                               bundle.scene.terrain_roi, config);
        if (!obs.xy.empty()) diag.terrain = model.recursive_update(obs);
      }
      diag.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
      record(k, diag, state.rotation, state.translation);
    }
  });
}

// One lm_solve on the reference (scan_matcher.cpp:257-358) with the wheel
// rows of two fixed-link legs (lever arms hL, hR; nullptr = no manifold).
// out: R9, t3; rep[8] = converged, failed, degenerate, outer, accepted,
// correspondences, final_cost, smallest eigenvalue; trace (cap) costs.
int ref_lm_solve(void* map, const double* px, const double* py, const double* pz, const unsigned char* kind,
                 size_t n, const double* R0, const double* t0, void* model, const double* hL, const double* hR,
                 double wheel_radius, const double* cfg, double lambda_M, double manifold_huber,
                 double* Rout, double* tout, double* rep, double* trace, size_t cap, size_t* ntrace) {
  return guarded([&] {
    const FeatureCloud f = to_cloud(px, py, pz, kind, nullptr, n);
    RobotState init;
    init.rotation = to_m3(R0);
    init.translation = Vec3(t0[0], t0[1], t0[2]);
    match::SolverConfig sc = to_solver(cfg);
    sc.lambda_manifold = lambda_M;
    sc.manifold_huber_delta = manifold_huber;
    JointConfig joints;
    kin::LegModel leg;
    match::ManifoldInputs mi;
    if (model && hL && hR) {
      leg.wheel_radius = wheel_radius;
      leg.left = fixed_chain(hL[0], hL[1], hL[2]);
      leg.right = fixed_chain(hR[0], hR[1], hR[2]);
      mi = {&joints, &leg, &M(model)->m};
    }
    match::SolveReport r;
    const RobotState out = match::lm_solve(init, f, *static_cast<match::LocalMap*>(map), mi, sc, &r);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) Rout[3 * i + j] = out.rotation(i, j);
    for (int i = 0; i < 3; ++i) tout[i] = out.translation(i);
    rep[0] = r.converged;
    rep[1] = r.failed;
    rep[2] = r.degenerate;
    rep[3] = r.outer_iterations;
    rep[4] = r.accepted_steps;
    rep[5] = static_cast<double>(r.correspondence_count);
    rep[6] = r.final_cost;
    rep[7] = r.smallest_feature_eigenvalue;
    *ntrace = r.cost_trace.size();
    for (size_t i = 0; i < r.cost_trace.size() && i < cap; ++i) trace[i] = r.cost_trace[i];
  });
}

}  // extern "C"
