// terralio_b200/terrain.hpp — the reference's C++ terrain API
// (proj/core/include/terralio/terrain/{kernel,center_select,terrain_model}.hpp,
// kinematics/contact.hpp) rebuilt on the C-ABI in terralio_gpu.h.
//
// Drop-in notes: same namespaces, class/function names, argument meaning and
// exception types; the Eigen types are replaced by the small value types
// below (x()/y()/z() accessors like Eigen's). TerrainModel is move-only like
// the reference's (terrain_model.hpp:95). All numerics run on the GPU; this
// header holds no arithmetic beyond parameter plumbing.
#pragma once

#include <cmath>
#include <fstream>
#include <cstdint>
#include <array>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../terralio_gpu.h"

namespace terralio {

struct Vec2 {
  double v[2] = {0.0, 0.0};
  Vec2() = default;
  Vec2(double x, double y) : v{x, y} {}
  double x() const { return v[0]; }
  double y() const { return v[1]; }
  double& x() { return v[0]; }
  double& y() { return v[1]; }
  double squaredNorm() const { return v[0] * v[0] + v[1] * v[1]; }
  bool allFinite() const { return std::isfinite(v[0]) && std::isfinite(v[1]); }
};

struct Vec3 {
  double v[3] = {0.0, 0.0, 0.0};
  Vec3() = default;
  Vec3(double x, double y, double z) : v{x, y, z} {}
  double x() const { return v[0]; }
  double y() const { return v[1]; }
  double z() const { return v[2]; }
};

// Row-major 3x3.
struct Mat3 {
  double a[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  double operator()(int r, int c) const { return a[3 * r + c]; }
  double& operator()(int r, int c) { return a[3 * r + c]; }
  static Mat3 Identity() { return Mat3{}; }
};

struct Rect {
  Vec2 min, max;
  bool contains(const Vec2& p) const {
    return p.x() >= min.x() && p.x() <= max.x() && p.y() >= min.y() && p.y() <= max.y();
  }
  Rect dilated(double m) const {
    return {{min.x() - m, min.y() - m}, {max.x() + m, max.y() + m}};
  }
};

namespace gpu {

// Maps a status code onto the reference's exception types.
struct NoSupportedCentersError;
[[noreturn]] void throw_status(tlg_status st);

inline void check(tlg_status st) {
  if (st != TLG_OK) throw_status(st);
}

// Process-wide default device context (device 0, private stream).
class Context {
 public:
  explicit Context(int device = 0, void* stream = nullptr) {
    check(tlg_ctx_create(device, stream, &ctx_));
  }
  ~Context() { tlg_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  tlg_ctx* get() const { return ctx_; }
  static Context& instance() {
    static Context c;
    return c;
  }

 private:
  tlg_ctx* ctx_ = nullptr;
};

}  // namespace gpu

namespace terrain {

// kernel.hpp:12-24
struct KernelParams {
  double sigma = 0.04;
  double sigma_eps = 0.1;
  double lambda = 1e-3;
  double cutoff_radius = 0.0;
  double sigma_tilde() const { return std::sqrt(sigma * sigma + sigma_eps * sigma_eps); }
  double moment_scale() const {
    const double st2 = sigma * sigma + sigma_eps * sigma_eps;
    return sigma * sigma / st2;
  }
  void finalize() {
    tlg_kernel_params p = c();
    gpu::check(tlg_kernel_finalize(&p));
    cutoff_radius = p.cutoff_radius;
  }
  tlg_kernel_params c() const { return {sigma, sigma_eps, lambda, cutoff_radius}; }
};

struct SparseVec {
  std::vector<std::pair<std::uint32_t, double>> entries;
};

// center_select.hpp:11-32
struct TerrainObservation {
  std::vector<Vec2> xy;
  std::vector<double> z;
  std::size_t size() const { return xy.size(); }
  void validate() const {
    if (xy.size() != z.size()) throw std::invalid_argument("observation xy/z length mismatch");
    if (xy.empty()) throw std::invalid_argument("empty observation");
    for (std::size_t i = 0; i < xy.size(); ++i)
      if (!xy[i].allFinite() || !std::isfinite(z[i]))
        throw std::invalid_argument("non-finite observation coordinate");
  }
};

struct CenterSet {
  std::vector<Vec2> centers;
  double mesh_resolution = 0.07;
  double accept_radius = 0.07;
  int accept_count = 3;
  Rect roi;
  tlg_center_params c() const {
    return {mesh_resolution, accept_radius, accept_count, 0,
            roi.min.x(),     roi.min.y(),   roi.max.x(), roi.max.y()};
  }
};

struct NoSupportedCenters : std::runtime_error {
  NoSupportedCenters() : std::runtime_error("no supported centers") {}
};

struct HeightQuery {
  double z = 0.0;
  bool supported = false;
};

struct UpdateReport {
  std::size_t active_blocks = 0, active_centers = 0, born_centers = 0;
  bool rejected = false;
};

namespace detail {
struct Soa {
  std::vector<double> x, y;
};
inline Soa split(const std::vector<Vec2>& v) {
  Soa s;
  s.x.resize(v.size());
  s.y.resize(v.size());
  for (std::size_t i = 0; i < v.size(); ++i) {
    s.x[i] = v[i].x();
    s.y[i] = v[i].y();
  }
  return s;
}
inline std::vector<Vec2> nodes(tlg_status (*fn)(tlg_ctx*, const double*, const double*,
                                                const double*, size_t, size_t, tlg_mem,
                                                const tlg_center_params*, double*, double*,
                                                size_t, size_t*, tlg_mem),
                               const TerrainObservation& pts, const tlg_center_params& cp) {
  const Soa s = split(pts.xy);
  size_t cap = std::max<size_t>(64, pts.size()), n = 0;
  std::vector<double> ox(cap), oy(cap);
  tlg_status st = fn(gpu::Context::instance().get(), s.x.data(), s.y.data(), pts.z.data(),
                     pts.xy.size(), pts.z.size(), TLG_HOST, &cp, ox.data(), oy.data(), cap, &n,
                     TLG_HOST);
  if (st == TLG_BUFFER_TOO_SMALL) {
    cap = n;
    ox.resize(cap);
    oy.resize(cap);
    st = fn(gpu::Context::instance().get(), s.x.data(), s.y.data(), pts.z.data(), pts.xy.size(),
            pts.z.size(), TLG_HOST, &cp, ox.data(), oy.data(), cap, &n, TLG_HOST);
  }
  gpu::check(st);
  std::vector<Vec2> out(n);
  for (size_t i = 0; i < n; ++i) out[i] = {ox[i], oy[i]};
  return out;
}
}  // namespace detail

// center_select.cpp:18-76
inline std::vector<Vec2> supported_mesh_nodes(const TerrainObservation& points, const Rect& roi,
                                              double mesh_resolution, double accept_radius,
                                              int accept_count) {
  CenterSet p;
  p.roi = roi;
  p.mesh_resolution = mesh_resolution;
  p.accept_radius = accept_radius;
  p.accept_count = accept_count;
  return detail::nodes(&tlg_supported_mesh_nodes, points, p.c());
}

inline CenterSet select_centers(const TerrainObservation& points, const Rect& roi,
                                double mesh_resolution, double accept_radius, int accept_count) {
  CenterSet set;
  set.roi = roi;
  set.mesh_resolution = mesh_resolution;
  set.accept_radius = accept_radius;
  set.accept_count = accept_count;
  set.centers = detail::nodes(&tlg_select_centers, points, set.c());
  return set;
}

// terrain_model.hpp:28-97 over a device-resident model
class TerrainModel {
 public:
  TerrainModel() = default;
  TerrainModel(KernelParams kernel, CenterSet centers) {
    const detail::Soa s = detail::split(centers.centers);
    const tlg_kernel_params k = kernel.c();
    const tlg_center_params cp = centers.c();
    tlg_model* m = nullptr;
    gpu::check(tlg_model_create(gpu::Context::instance().get(), &k, &cp, s.x.data(), s.y.data(),
                                s.x.size(), TLG_HOST, &m));
    m_.reset(m);
  }
  explicit TerrainModel(tlg_model* adopt) : m_(adopt) {}
  TerrainModel(TerrainModel&&) = default;
  TerrainModel& operator=(TerrainModel&&) = default;

  KernelParams kernel() const {
    tlg_kernel_params k;
    gpu::check(tlg_model_kernel(m_.get(), &k));
    return {k.sigma, k.sigma_eps, k.lambda, k.cutoff_radius};
  }
  CenterSet centers() const {
    tlg_center_params p;
    gpu::check(tlg_model_center_params(m_.get(), &p));
    CenterSet s;
    s.mesh_resolution = p.mesh_resolution;
    s.accept_radius = p.accept_radius;
    s.accept_count = p.accept_count;
    s.roi = {{p.roi_min_x, p.roi_min_y}, {p.roi_max_x, p.roi_max_y}};
    const std::size_t n = num_centers();
    std::vector<double> x(n), y(n);
    gpu::check(tlg_model_get_centers(m_.get(), x.data(), y.data(), TLG_HOST));
    s.centers.resize(n);
    for (std::size_t i = 0; i < n; ++i) s.centers[i] = {x[i], y[i]};
    return s;
  }
  // host mirror, read from the device once per model change (not per call)
  const std::vector<double>& weights() const {
    if (w_at_ != ver_) {
      w_.resize(num_centers());
      if (!w_.empty()) gpu::check(tlg_model_get_weights(m_.get(), w_.data(), TLG_HOST));
      w_at_ = ver_;
    }
    return w_;
  }
  std::size_t num_centers() const {
    size_t n = 0, b = 0;
    gpu::check(tlg_model_counts(m_.get(), &n, &b));
    return n;
  }
  std::size_t num_blocks() const {
    size_t n = 0, b = 0;
    gpu::check(tlg_model_counts(m_.get(), &n, &b));
    return b;
  }
  std::uint32_t block_of(std::uint32_t center) const {
    if (bidx_at_ != ver_) {
      bidx_.resize(num_centers());
      if (!bidx_.empty()) gpu::check(tlg_model_get_block_index(m_.get(), bidx_.data(), TLG_HOST));
      bidx_at_ = ver_;
    }
    return bidx_.at(center);
  }
  std::vector<std::uint32_t> block_members(std::uint32_t b) const {
    size_t n = 0;
    gpu::check(tlg_model_block_size(m_.get(), b, &n));
    std::vector<std::uint32_t> out(n);
    gpu::check(tlg_model_get_block_members(m_.get(), b, out.data()));
    return out;
  }
  // column-major bn x bn (Eigen::MatrixXd storage order)
  std::vector<double> block_info_inverse(std::uint32_t b) const {
    size_t n = 0;
    gpu::check(tlg_model_block_size(m_.get(), b, &n));
    std::vector<double> out(n * n);
    if (n) gpu::check(tlg_model_get_block_info_inverse(m_.get(), b, out.data(), TLG_HOST));
    return out;
  }

  // terrain_model.cpp:97-107
  SparseVec moment_feature(const Vec2& x) const {
    uint32_t rp[2];
    std::vector<uint32_t> ids(4096);
    std::vector<double> vals(4096);
    size_t nnz = 0;
    gpu::check(tlg_moment_features(m_.get(), &x.v[0], &x.v[1], 1, TLG_HOST, rp, ids.data(),
                                   vals.data(), ids.size(), &nnz, TLG_HOST));
    SparseVec out;
    for (size_t i = 0; i < nnz; ++i) out.entries.emplace_back(ids[i], vals[i]);
    return out;
  }

  // terrain_model.cpp:109-143 (a query of one point; batch with predict())
  HeightQuery predict_height(const Vec2& x) const {
    double z = 0.0;
    uint8_t s = 0;
    gpu::check(tlg_eval(m_.get(), &x.v[0], &x.v[1], 1, TLG_HOST, &z, &s, nullptr, nullptr,
                        TLG_HOST));
    return {z, s != 0};
  }
  // height, support flag and gradient of one point in one device call
  HeightQuery predict_height_gradient(const Vec2& x, Vec2* grad) const {
    double z = 0.0;
    uint8_t s = 0;
    Vec2 g;
    gpu::check(tlg_eval(m_.get(), &x.v[0], &x.v[1], 1, TLG_HOST, &z, &s, &g.v[0], &g.v[1], TLG_HOST));
    if (grad) *grad = g;
    return {z, s != 0};
  }
  Vec2 predict_gradient(const Vec2& x) const {
    Vec2 g;
    gpu::check(tlg_eval(m_.get(), &x.v[0], &x.v[1], 1, TLG_HOST, nullptr, nullptr, &g.v[0],
                        &g.v[1], TLG_HOST));
    return g;
  }
  // Batched: SoA host arrays; any output may be null.
  void predict(const double* x, const double* y, std::size_t n, double* z, uint8_t* supported,
               double* gx, double* gy) const {
    gpu::check(tlg_eval(m_.get(), x, y, n, TLG_HOST, z, supported, gx, gy, TLG_HOST));
  }

  // terrain_model.cpp:145-253
  UpdateReport recursive_update(const TerrainObservation& obs, bool allow_birth = true) {
    const detail::Soa s = detail::split(obs.xy);
    tlg_update_report r{};
    const tlg_status st = tlg_recursive_update(m_.get(), s.x.data(), s.y.data(), obs.z.data(),
                                               obs.xy.size(), obs.z.size(), TLG_HOST,
                                               allow_birth ? 1 : 0, &r);
    ++ver_;  // births may have landed even when the call throws
    gpu::check(st);
    return {static_cast<std::size_t>(r.active_blocks), static_cast<std::size_t>(r.active_centers),
            static_cast<std::size_t>(r.born_centers), r.rejected != 0};
  }

  // terrain_model.cpp:255-267: the reference's grid walk, one batched device
  // evaluation, ostream default formatting
  void export_csv(const std::string& path, double grid_step) const {
    tlg_center_params cp{};
    gpu::check(tlg_model_center_params(m_.get(), &cp));
    std::vector<double> xs, ys;
    for (double x = cp.roi_min_x; x <= cp.roi_max_x + 1e-12; x += grid_step)
      for (double y = cp.roi_min_y; y <= cp.roi_max_y + 1e-12; y += grid_step) {
        xs.push_back(x);
        ys.push_back(y);
      }
    std::vector<double> z(xs.size());
    std::vector<uint8_t> s(xs.size());
    if (!xs.empty()) predict(xs.data(), ys.data(), xs.size(), z.data(), s.data(), nullptr, nullptr);
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot open " + path);
    out << "x,y,z_pred\n";
    for (std::size_t i = 0; i < xs.size(); ++i)
      if (s[i]) out << xs[i] << ',' << ys[i] << ',' << z[i] << '\n';
  }

  // Point-sharded fit_batch_ridge (tlg_batch_ridge_*): H (elems
  // doubles) and b (n) are DEVICE buffers sized from batch_system().
  struct BatchSystem {
    std::size_t n = 0, ld = 0, elems = 0;
  };
  BatchSystem batch_system() const {
    BatchSystem s;
    gpu::check(tlg_batch_ridge_system(m_.get(), &s.n, &s.ld, &s.elems));
    return s;
  }
  void batch_assemble(const TerrainObservation& shard, double* H, double* b, bool add_lambda) {
    const detail::Soa o = detail::split(shard.xy);
    const BatchSystem s = batch_system();
    gpu::check(tlg_batch_ridge_assemble(m_.get(), o.x.data(), o.y.data(), shard.z.data(),
                                        shard.xy.size(), TLG_HOST, H, s.ld, b,
                                        add_lambda ? 1 : 0));
  }
  void batch_solve(double* H, double* b) {
    gpu::check(tlg_batch_ridge_solve(m_.get(), H, batch_system().ld, b));
    ++ver_;
  }
  // kernel_eval's exact per-pair cutoff test everywhere (tlg_model_set_exact_cutoff)
  void set_exact_cutoff(bool exact) {
    gpu::check(tlg_model_set_exact_cutoff(m_.get(), exact ? 1 : 0));
  }

  void save(const std::string& path) const { gpu::check(tlg_model_save(m_.get(), path.c_str())); }
  static TerrainModel load(const std::string& path) {
    tlg_model* m = nullptr;
    gpu::check(tlg_model_load(gpu::Context::instance().get(), path.c_str(), &m));
    return TerrainModel(m);
  }

  tlg_model* handle() const { return m_.get(); }
  // the host mirrors are stale after changes made through handle()
  void invalidate() { ++ver_; }
  tlg_model* get() const { return m_.get(); }

 private:
  struct Del {
    void operator()(tlg_model* m) const { tlg_model_destroy(m); }
  };
  std::unique_ptr<tlg_model, Del> m_;
  std::uint64_t ver_ = 1;
  mutable std::vector<double> w_;
  mutable std::uint64_t w_at_ = 0;
  mutable std::vector<std::uint32_t> bidx_;
  mutable std::uint64_t bidx_at_ = 0;
};

// terrain_model.cpp:269-308
inline TerrainModel fit_batch_ridge(const KernelParams& params, const CenterSet& centers,
                                    const TerrainObservation& obs) {
  const detail::Soa c = detail::split(centers.centers);
  const detail::Soa o = detail::split(obs.xy);
  const tlg_kernel_params k = params.c();
  const tlg_center_params cp = centers.c();
  tlg_model* m = nullptr;
  gpu::check(tlg_fit_batch_ridge(gpu::Context::instance().get(), &k, &cp, c.x.data(), c.y.data(),
                                 c.x.size(), o.x.data(), o.y.data(), obs.z.data(), obs.xy.size(),
                                 obs.z.size(), TLG_HOST, &m));
  return TerrainModel(m);
}

// Point-sharded fit_batch_ridge: every rank holds `model` built from the
// same centres and its shard of the observations; allreduce_sum(ptr, count)
// sums a device buffer over the ranks in place (e.g. ncclAllReduce + a
// stream synchronize). Exactly one rank passes root = true (adds lambda I).
template <class AllReduce>
void fit_batch_ridge_sharded(TerrainModel& model, const TerrainObservation& shard, bool root,
                             double* H, double* b, AllReduce&& allreduce_sum) {
  const TerrainModel::BatchSystem s = model.batch_system();
  model.batch_assemble(shard, H, b, root);
  allreduce_sum(H, s.elems);
  allreduce_sum(b, s.n);
  model.batch_solve(H, b);
}

// The library's own communicator (tlg_comm, one process per GPU): rank 0
// makes the id (unique_id()), the job broadcasts it, every rank constructs.
class Communicator {
 public:
  using Id = std::array<unsigned char, TLG_COMM_ID_BYTES>;
  static Id unique_id() {
    Id id{};
    gpu::check(tlg_comm_unique_id(id.data()));
    return id;
  }
  Communicator(const Id& id, int rank, int size) {
    tlg_comm* c = nullptr;
    gpu::check(tlg_comm_init(gpu::Context::instance().get(), id.data(), rank, size, &c));
    c_.reset(c);
  }
  tlg_comm* get() const { return c_.get(); }

 private:
  struct Del {
    void operator()(tlg_comm* c) const { tlg_comm_destroy(c); }
  };
  std::unique_ptr<tlg_comm, Del> c_;
};

// fit_batch_ridge over point shards through the library communicator: the
// packed structural nonzeros of the partial systems and the rhs are reduced
// (NCCL), every rank solves and ends with the same model.
inline void fit_batch_ridge_sharded(TerrainModel& model, const Communicator& comm,
                                    const TerrainObservation& shard) {
  const detail::Soa o = detail::split(shard.xy);
  gpu::check(tlg_fit_batch_ridge_sharded(model.get(), comm.get(), o.x.data(), o.y.data(),
                                         shard.z.data(), shard.xy.size(), TLG_HOST));
  model.invalidate();
}

}  // namespace terrain

namespace eval {

// metrics.hpp:42-51
struct Histogram {
  std::vector<double> edges;
  std::vector<std::size_t> counts;
  std::size_t trimmed = 0;
  std::size_t overflow = 0;
  std::size_t total() const {
    std::size_t n = overflow;
    for (const std::size_t c : counts) n += c;
    return n;
  }
  double fraction_below(double threshold) const {
    const std::size_t n = total();
    if (n == 0) return 0.0;
    std::size_t below = 0;
    for (std::size_t b = 0; b < counts.size(); ++b)
      if (edges[b + 1] <= threshold + 1e-12) below += counts[b];
    return static_cast<double>(below) / static_cast<double>(n);
  }
};

// metrics.cpp:199-232
inline Histogram terrain_error_histogram(const terrain::TerrainModel& model,
                                         const std::vector<Vec2>& xy, const std::vector<double>& z,
                                         double trim_fraction, int bins) {
  if (xy.empty() || xy.size() != z.size())
    throw std::invalid_argument("histogram needs matched non-empty samples");
  std::vector<double> x(xy.size()), y(xy.size());
  for (std::size_t i = 0; i < xy.size(); ++i) {
    x[i] = xy[i].x();
    y[i] = xy[i].y();
  }
  Histogram h;
  h.edges.resize(bins + 1);
  std::vector<uint64_t> c(bins > 0 ? bins : 1);
  uint64_t tr = 0, ov = 0;
  gpu::check(tlg_terrain_error_histogram(model.handle(), x.data(), y.data(), z.data(), xy.size(),
                                         TLG_HOST, trim_fraction, bins, h.edges.data(), c.data(),
                                         &tr, &ov));
  h.counts.assign(c.begin(), c.begin() + bins);
  h.trimmed = tr;
  h.overflow = ov;
  return h;
}

}  // namespace eval

namespace match {

// types.hpp:36-42 / FeatureCloud
enum class FeatureKind : uint8_t { Edge = 0, Planar = 1, Ground = 2 };
struct FeaturePoint {
  Vec3 p;
  FeatureKind kind = FeatureKind::Planar;
  int32_t label = -1;
};
struct FeatureCloud {
  double timestamp = 0.0;
  std::vector<FeaturePoint> points;
};

// The association fields of SolverConfig (scan_matcher.hpp:15-49) + LM knobs.
struct SolverConfig {
  double lambda_manifold = 1.0, lm_init_damping = 1e-4;
  int lm_max_iters = 10, lm_max_inner = 8, lm_max_rejects = 12;
  double tol_dcost = 1e-10, tol_dstate = 1e-10, corr_gate = 1.0;
  int min_correspondences = 10;
  double huber_delta = 0.1, manifold_huber_delta = 0.05, plane_fit_tol = 0.025,
         plane_eig_ratio = 5.0, edge_eig_ratio = 3.0, edge_fit_tol = 0.05, edge_min_extent = 0.05,
         degeneracy_eig_min = 10.0, trim_ratio = 5.0, trim_floor = 0.003,
         ground_corr_voxel = 0.25, ground_corr_radius = 4.0;
  tlg_match_config c() const {
    return {corr_gate,      huber_delta, plane_fit_tol, plane_eig_ratio,   edge_eig_ratio,
            edge_fit_tol,   edge_min_extent, trim_ratio, trim_floor, ground_corr_voxel,
            ground_corr_radius};
  }
};

struct MapConfig {
  double voxel_size = 0.1;
  std::size_t window = 20;
};

namespace detail {
struct Soa3 {
  std::vector<double> x, y, z;
  std::vector<uint8_t> kind;
  std::vector<int32_t> label;
};
inline Soa3 split(const FeatureCloud& f) {
  Soa3 s;
  for (const auto& p : f.points) {
    s.x.push_back(p.p.x());
    s.y.push_back(p.p.y());
    s.z.push_back(p.p.z());
    s.kind.push_back(static_cast<uint8_t>(p.kind));
    s.label.push_back(p.label);
  }
  return s;
}
}  // namespace detail

// local_map.hpp:17-50 (the kd-trees are device-side uniform grids)
class LocalMap {
 public:
  explicit LocalMap(MapConfig config = {}) {
    tlg_map* m = nullptr;
    gpu::check(tlg_map_create(gpu::Context::instance().get(), config.voxel_size, config.window,
                              &m));
    m_.reset(m);
  }
  void insert(const FeatureCloud& scan, const Mat3& rotation, const Vec3& translation) {
    const detail::Soa3 s = detail::split(scan);
    gpu::check(tlg_map_insert(m_.get(), s.x.data(), s.y.data(), s.z.data(), s.kind.data(),
                              s.label.data(), s.x.size(), TLG_HOST, rotation.a, translation.v));
  }
  std::size_t size() const { return count(0) + count(1); }
  bool empty() const { return size() == 0; }
  tlg_map* handle() const { return m_.get(); }

 private:
  std::size_t count(int kind) const {
    std::size_t n = 0;
    gpu::check(tlg_map_points(m_.get(), kind, nullptr, nullptr, 0, &n));
    return n;
  }
  struct Del {
    void operator()(tlg_map* m) const { tlg_map_destroy(m); }
  };
  std::unique_ptr<tlg_map, Del> m_;
};

struct Correspondence {  // scan_matcher.hpp:51-58
  FeatureKind kind = FeatureKind::Edge;
  Vec3 p_sensor;
  Vec3 line_point, line_direction{1.0, 0.0, 0.0}, plane_normal{0.0, 0.0, 1.0};
  double plane_offset = 0.0, weight = 1.0;
  int32_t map_label = -1;
};

// scan_matcher.cpp:44-183 at the pose (R, t); the device keeps the result for
// feature_normal_eq
inline std::vector<Correspondence> build_correspondences(const FeatureCloud& features,
                                                         const Mat3& R, const Vec3& t,
                                                         const LocalMap& map,
                                                         const SolverConfig& config) {
  const detail::Soa3 s = detail::split(features);
  const tlg_match_config c = config.c();
  std::size_t n = 0;
  gpu::check(tlg_build_correspondences(map.handle(), s.x.data(), s.y.data(), s.z.data(),
                                       s.kind.data(), s.x.size(), TLG_HOST, R.a, t.v, &c, &n));
  std::vector<int32_t> kind(n), label(n);
  std::vector<uint32_t> feat(n);
  std::vector<double> par(7 * n), w(n);
  gpu::check(tlg_correspondences_get(map.handle(), kind.data(), feat.data(), par.data(), w.data(),
                                     label.data(), nullptr, nullptr, n));
  std::vector<Correspondence> out(n);
  for (std::size_t i = 0; i < n; ++i) {
    auto& o = out[i];
    const double* p = &par[7 * i];
    o.kind = kind[i] == 0 ? FeatureKind::Edge : FeatureKind::Planar;
    o.p_sensor = features.points[feat[i]].p;
    if (kind[i] == 0) {
      o.line_point = {p[0], p[1], p[2]};
      o.line_direction = {p[3], p[4], p[5]};
    } else {
      o.plane_normal = {p[0], p[1], p[2]};
      o.plane_offset = p[3];
    }
    o.weight = w[i];
    o.map_label = label[i];
  }
  return out;
}

// feature rows of total_cost (scan_matcher.cpp:185-216) for the map's last
// correspondences, reduced to the normal equations
inline tlg_normal_eq feature_normal_eq(const LocalMap& map, const Mat3& R, const Vec3& t) {
  tlg_normal_eq ne{};
  gpu::check(tlg_feature_normal_eq(map.handle(), R.a, t.v, &ne));
  return ne;
}

// scan_matcher.cpp:300-305
inline bool lm_step(const tlg_normal_eq& ne, double mu, double delta[6]) {
  return tlg_lm_step(gpu::Context::instance().get(), &ne, mu, delta) == TLG_OK;
}

}  // namespace match

namespace kin {

// Batched manifold rows (contact.cpp:7-39 + scan_matcher.cpp:221-248) and the
// fused normal equations (scan_matcher.cpp:296-299).
struct ManifoldRows {
  std::vector<double> r, J;  // J column-major rows x 6 (Eigen CostEval layout)
  std::vector<uint8_t> valid;
  tlg_normal_eq ne{};
};

inline ManifoldRows manifold_rows(const terrain::TerrainModel& terrain, const Mat3& R,
                                  const Vec3& t, const std::vector<Vec3>& lever,
                                  double wheel_radius, double lambda_M, double huber_delta) {
  const std::size_t n = lever.size();
  std::vector<double> hx(n), hy(n), hz(n);
  for (std::size_t i = 0; i < n; ++i) {
    hx[i] = lever[i].x();
    hy[i] = lever[i].y();
    hz[i] = lever[i].z();
  }
  ManifoldRows out;
  out.r.resize(n);
  out.J.resize(6 * n);
  out.valid.resize(n);
  gpu::check(tlg_manifold_rows(terrain.handle(), R.a, t.v, hx.data(), hy.data(), hz.data(), n,
                               TLG_HOST, wheel_radius, lambda_M, huber_delta, out.r.data(),
                               out.J.data(), out.valid.data(), nullptr, TLG_HOST, &out.ne));
  return out;
}

struct ManifoldResidual {
  double value = 0.0;
  bool valid = false;
};

// contact.cpp:7-19 for one wheel with lever arm h (chain_end_position(q)).
inline ManifoldResidual manifold_residual(const Mat3& R, const Vec3& t, const Vec3& h,
                                          double wheel_radius,
                                          const terrain::TerrainModel& terrain) {
  double raw = 0.0;
  uint8_t valid = 0;
  gpu::check(tlg_manifold_rows(terrain.handle(), R.a, t.v, &h.v[0], &h.v[1], &h.v[2], 1,
                               TLG_HOST, wheel_radius, 1.0, 0.0, nullptr, nullptr, &valid, &raw,
                               TLG_HOST, nullptr));
  return {valid ? raw : 0.0, valid != 0};
}

}  // namespace kin

namespace gpu {
[[noreturn]] inline void throw_status(tlg_status st) {
  const std::string msg = tlg_last_error();
  switch (st) {
    case TLG_INVALID_ARGUMENT:
      throw std::invalid_argument(msg);
    case TLG_DOMAIN_ERROR:
      throw std::domain_error(msg);
    case TLG_NO_SUPPORTED_CENTERS:
      throw terrain::NoSupportedCenters();
    case TLG_OUT_OF_MEMORY:
      throw std::bad_alloc();
    default:
      throw std::runtime_error(msg);
  }
}
}  // namespace gpu

}  // namespace terralio
