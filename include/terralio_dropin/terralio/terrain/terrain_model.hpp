// terralio drop-in: proj/core/include/terralio/terrain/terrain_model.hpp:16-103
// over a device-resident model (tlg_model). Same public API, including the
// reference's reference-returning accessors: weights(), centers(),
// block_members(b) and block_info_inverse(b) return host mirrors that are
// refreshed lazily — once per model change, not per call — so loops such as
// `for j: model.weights()(j)` cost one device read in total. Move-only like
// the reference's (terrain_model.hpp:95).
#pragma once

#include <Eigen/Core>
#include <cstdint>
#include <fstream>
#include <memory>
#include <string>
#include <vector>

#include "terralio/detail/device.hpp"
#include "terralio/terrain/center_select.hpp"
#include "terralio/terrain/kernel.hpp"
#include "terralio/types.hpp"

namespace terralio::terrain {

struct HeightQuery {
  double z = 0.0;
  bool supported = false;
};

struct UpdateReport {
  std::size_t active_blocks = 0;
  std::size_t active_centers = 0;
  std::size_t born_centers = 0;
  bool rejected = false;
};

class TerrainModel {
 public:
  TerrainModel() = default;
  TerrainModel(KernelParams kernel, CenterSet centers) {
    kernel.finalize();
    const detail::XY c(centers.centers);
    const tlg_kernel_params k = kernel.c_params();
    const tlg_center_params cp = centers.c_params();
    tlg_model* m = nullptr;
    ::terralio::detail::tlg_check(tlg_model_create(::terralio::detail::Device::ctx(), &k, &cp, c.x.data(),
                                                   c.y.data(), c.x.size(), TLG_HOST, &m));
    adopt(m);
  }
  explicit TerrainModel(tlg_model* m) { adopt(m); }
  TerrainModel(TerrainModel&&) = default;
  TerrainModel& operator=(TerrainModel&&) = default;
  TerrainModel(const TerrainModel&) = delete;
  TerrainModel& operator=(const TerrainModel&) = delete;

  const KernelParams& kernel() const { return mirror_->kernel; }
  const CenterSet& centers() const {
    refresh_centers();
    return mirror_->centers;
  }
  const Eigen::VectorXd& weights() const {
    if (mirror_->weights_at != mirror_->version) {
      const std::size_t n = num_centers();
      mirror_->weights.resize(static_cast<Eigen::Index>(n));
      if (n) ::terralio::detail::tlg_check(tlg_model_get_weights(m_.get(), mirror_->weights.data(), TLG_HOST));
      mirror_->weights_at = mirror_->version;
    }
    return mirror_->weights;
  }
  std::size_t num_centers() const {
    if (!m_) return 0;
    size_t n = 0, b = 0;
    ::terralio::detail::tlg_check(tlg_model_counts(m_.get(), &n, &b));
    return n;
  }
  std::size_t num_blocks() const {
    if (!m_) return 0;
    size_t n = 0, b = 0;
    ::terralio::detail::tlg_check(tlg_model_counts(m_.get(), &n, &b));
    return b;
  }
  std::uint32_t block_of(std::uint32_t center) const {
    refresh_structure();
    return mirror_->block_index[center];
  }
  const std::vector<std::uint32_t>& block_members(std::uint32_t b) const {
    refresh_structure();
    return mirror_->members[b];
  }
  const Eigen::MatrixXd& block_info_inverse(std::uint32_t b) const {
    refresh_structure();
    auto& slot = mirror_->info_inv[b];
    if (mirror_->info_at[b] != mirror_->version) {
      const auto bn = static_cast<Eigen::Index>(mirror_->members[b].size());
      slot.resize(bn, bn);
      if (bn)
        ::terralio::detail::tlg_check(tlg_model_get_block_info_inverse(m_.get(), b, slot.data(), TLG_HOST));
      mirror_->info_at[b] = mirror_->version;
    }
    return slot;
  }

  // terrain_model.cpp:97-107
  SparseVec moment_feature(const Vec2& x) const {
    SparseVec out;
    if (!m_) return out;
    const double qx = x.x(), qy = x.y();
    uint32_t rp[2] = {0, 0};
    std::vector<uint32_t> ids(256);
    std::vector<double> vals(256);
    size_t nnz = 0;
    tlg_status st = tlg_moment_features(m_.get(), &qx, &qy, 1, TLG_HOST, rp, ids.data(), vals.data(),
                                        ids.size(), &nnz, TLG_HOST);
    if (st == TLG_BUFFER_TOO_SMALL) {
      ids.resize(nnz);
      vals.resize(nnz);
      st = tlg_moment_features(m_.get(), &qx, &qy, 1, TLG_HOST, rp, ids.data(), vals.data(), ids.size(),
                               &nnz, TLG_HOST);
    }
    ::terralio::detail::tlg_check(st);
    out.entries.reserve(nnz);
    for (size_t i = 0; i < nnz; ++i) out.entries.emplace_back(ids[i], vals[i]);
    return out;
  }

  // terrain_model.cpp:109-143, one query (batch callers: predict())
  HeightQuery predict_height(const Vec2& x) const {
    if (!m_) return {};
    const double qx = x.x(), qy = x.y();
    double z = 0.0;
    uint8_t s = 0;
    ::terralio::detail::tlg_check(tlg_eval(m_.get(), &qx, &qy, 1, TLG_HOST, &z, &s, nullptr, nullptr, TLG_HOST));
    return {z, s != 0};
  }
  Vec2 predict_gradient(const Vec2& x) const {
    if (!m_) return Vec2::Zero();
    const double qx = x.x(), qy = x.y();
    double gx = 0.0, gy = 0.0;
    ::terralio::detail::tlg_check(tlg_eval(m_.get(), &qx, &qy, 1, TLG_HOST, nullptr, nullptr, &gx, &gy, TLG_HOST));
    return Vec2(gx, gy);
  }
  // Batched height / supported / gradient over SoA host arrays (any output
  // may be null): one device evaluation for n points.
  void predict(const double* x, const double* y, std::size_t n, double* z, uint8_t* supported, double* gx,
               double* gy) const {
    ::terralio::detail::tlg_check(tlg_eval(m_.get(), x, y, n, TLG_HOST, z, supported, gx, gy, TLG_HOST));
  }

  // terrain_model.cpp:145-253
  UpdateReport recursive_update(const TerrainObservation& obs, bool allow_birth = true) {
    const detail::XY s(obs.xy);
    tlg_update_report r{};
    const tlg_status st = tlg_recursive_update(m_.get(), s.x.data(), s.y.data(), obs.z.data(), obs.xy.size(),
                                               obs.z.size(), TLG_HOST, allow_birth ? 1 : 0, &r);
    ++mirror_->version;  // births may have landed even if the call throws
    ::terralio::detail::tlg_check(st);
    return {static_cast<std::size_t>(r.active_blocks), static_cast<std::size_t>(r.active_centers),
            static_cast<std::size_t>(r.born_centers), r.rejected != 0};
  }

  // terrain_model.cpp:255-267: the reference's grid walk, one batched device
  // evaluation, default ostream formatting
  void export_csv(const std::string& path, double grid_step) const {
    const Rect& roi = mirror_->roi;
    std::vector<double> xs, ys;
    for (double x = roi.min.x(); x <= roi.max.x() + 1e-12; x += grid_step)
      for (double y = roi.min.y(); y <= roi.max.y() + 1e-12; y += grid_step) {
        xs.push_back(x);
        ys.push_back(y);
      }
    std::vector<double> z(xs.size());
    std::vector<uint8_t> sup(xs.size());
    if (!xs.empty()) predict(xs.data(), ys.data(), xs.size(), z.data(), sup.data(), nullptr, nullptr);
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot open " + path);
    out << "x,y,z_pred\n";
    for (std::size_t i = 0; i < xs.size(); ++i)
      if (sup[i]) out << xs[i] << ',' << ys[i] << ',' << z[i] << '\n';
  }

  void save(const std::string& path) const {
    ::terralio::detail::tlg_check(tlg_model_save(m_.get(), path.c_str()));
  }
  static TerrainModel load(const std::string& path) {
    tlg_model* m = nullptr;
    ::terralio::detail::tlg_check(tlg_model_load(::terralio::detail::Device::ctx(), path.c_str(), &m));
    return TerrainModel(m);
  }

  tlg_model* handle() const { return m_.get(); }
  // the host mirrors are stale after a change made through handle()
  void invalidate() { ++mirror_->version; }

 private:
  struct Mirror {
    KernelParams kernel;
    Rect roi;
    double mesh_resolution = 0.07, accept_radius = 0.07;
    int accept_count = 3;
    std::uint64_t version = 1;
    CenterSet centers;
    std::uint64_t centers_at = 0;
    Eigen::VectorXd weights;
    std::uint64_t weights_at = 0;
    std::vector<std::uint32_t> block_index;
    std::vector<std::vector<std::uint32_t>> members;
    std::vector<Eigen::MatrixXd> info_inv;
    std::vector<std::uint64_t> info_at;
    std::uint64_t structure_at = 0;
  };
  struct Del {
    void operator()(tlg_model* m) const { tlg_model_destroy(m); }
  };

  void adopt(tlg_model* m) {
    m_.reset(m);
    mirror_ = std::make_unique<Mirror>();
    tlg_kernel_params k{};
    ::terralio::detail::tlg_check(tlg_model_kernel(m, &k));
    mirror_->kernel = {k.sigma, k.sigma_eps, k.lambda, k.cutoff_radius};
    tlg_center_params p{};
    ::terralio::detail::tlg_check(tlg_model_center_params(m, &p));
    mirror_->roi = {Vec2(p.roi_min_x, p.roi_min_y), Vec2(p.roi_max_x, p.roi_max_y)};
    mirror_->mesh_resolution = p.mesh_resolution;
    mirror_->accept_radius = p.accept_radius;
    mirror_->accept_count = p.accept_count;
  }
  void refresh_centers() const {
    Mirror& r = *mirror_;
    if (r.centers_at == r.version) return;
    r.centers.mesh_resolution = r.mesh_resolution;
    r.centers.accept_radius = r.accept_radius;
    r.centers.accept_count = r.accept_count;
    r.centers.roi = r.roi;
    const std::size_t n = num_centers();
    std::vector<double> x(n), y(n);
    if (n) ::terralio::detail::tlg_check(tlg_model_get_centers(m_.get(), x.data(), y.data(), TLG_HOST));
    r.centers.centers.resize(n);
    for (std::size_t i = 0; i < n; ++i) r.centers.centers[i] = Vec2(x[i], y[i]);
    r.centers_at = r.version;
  }
  void refresh_structure() const {
    Mirror& r = *mirror_;
    if (r.structure_at == r.version) return;
    const std::size_t n = num_centers(), nb = num_blocks();
    r.block_index.resize(n);
    if (n) ::terralio::detail::tlg_check(tlg_model_get_block_index(m_.get(), r.block_index.data(), TLG_HOST));
    r.members.resize(nb);
    for (std::uint32_t b = 0; b < nb; ++b) {
      size_t bn = 0;
      ::terralio::detail::tlg_check(tlg_model_block_size(m_.get(), b, &bn));
      r.members[b].resize(bn);
      if (bn) ::terralio::detail::tlg_check(tlg_model_get_block_members(m_.get(), b, r.members[b].data()));
    }
    r.info_inv.resize(nb);
    r.info_at.assign(nb, 0);
    r.structure_at = r.version;
  }

  std::unique_ptr<tlg_model, Del> m_;
  std::unique_ptr<Mirror> mirror_ = std::make_unique<Mirror>();
};

// terrain_model.cpp:269-308 (std::runtime_error with a condition estimate on
// solver failure, from the device factorisation)
inline TerrainModel fit_batch_ridge(const KernelParams& params, const CenterSet& centers,
                                    const TerrainObservation& obs) {
  const detail::XY c(centers.centers);
  const detail::XY o(obs.xy);
  KernelParams k = params;
  k.finalize();
  const tlg_kernel_params kp = k.c_params();
  const tlg_center_params cp = centers.c_params();
  tlg_model* m = nullptr;
  ::terralio::detail::tlg_check(tlg_fit_batch_ridge(::terralio::detail::Device::ctx(), &kp, &cp, c.x.data(),
                                                    c.y.data(), c.x.size(), o.x.data(), o.y.data(), obs.z.data(),
                                                    obs.xy.size(), obs.z.size(), TLG_HOST, &m));
  return TerrainModel(m);
}

}  // namespace terralio::terrain
