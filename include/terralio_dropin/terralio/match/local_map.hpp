// terralio drop-in: proj/core/include/terralio/match/local_map.hpp:12-50.
// The sliding window of world-frame features lives on the device
// (tlg_map_*: voxel-thinned insert, per-kind uniform grids for the exact
// kNN); the reference's host kd-trees (edge_tree / planar_tree) have no
// counterpart — association runs on the device (build_correspondences).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "terralio/detail/device.hpp"
#include "terralio/types.hpp"

namespace terralio::match {

struct MapConfig {
  double voxel_size = 0.1;
  std::size_t window = 20;
};

class LocalMap {
 public:
  explicit LocalMap(MapConfig config = {}) {
    tlg_map* m = nullptr;
    ::terralio::detail::tlg_check(tlg_map_create(::terralio::detail::Device::ctx(), config.voxel_size,
                                                 config.window, &m));
    m_.reset(m);
  }
  void insert(const FeatureCloud& scan, const Mat3& rotation, const Vec3& translation) {
    const std::size_t n = scan.points.size();
    std::vector<double> x(n), y(n), z(n);
    std::vector<uint8_t> k(n);
    std::vector<int32_t> l(n);
    for (std::size_t i = 0; i < n; ++i) {
      x[i] = scan.points[i].p.x();
      y[i] = scan.points[i].p.y();
      z[i] = scan.points[i].p.z();
      k[i] = static_cast<uint8_t>(scan.points[i].kind);
      l[i] = scan.points[i].label;
    }
    double R[9], t[3] = {translation.x(), translation.y(), translation.z()};
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) R[3 * i + j] = rotation(i, j);
    ::terralio::detail::tlg_check(
        tlg_map_insert(m_.get(), x.data(), y.data(), z.data(), k.data(), l.data(), n, TLG_HOST, R, t));
  }
  bool empty() const { return size() == 0; }
  std::size_t size() const { return count(0) + count(1); }
  tlg_map* handle() const { return m_.get(); }

 private:
  std::size_t count(int kind) const {
    std::size_t n = 0;
    ::terralio::detail::tlg_check(tlg_map_points(m_.get(), kind, nullptr, nullptr, 0, &n));
    return n;
  }
  struct Del {
    void operator()(tlg_map* m) const { tlg_map_destroy(m); }
  };
  std::unique_ptr<tlg_map, Del> m_;
};

}  // namespace terralio::match
