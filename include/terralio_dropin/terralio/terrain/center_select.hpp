// terralio drop-in: proj/core/include/terralio/terrain/center_select.hpp:11-45
// on the device (tlg_supported_mesh_nodes / tlg_select_centers: node lists
// bit-identical to the reference's, in its i-outer, j-inner order).
#pragma once

#include <cmath>
#include <stdexcept>
#include <vector>

#include "terralio/detail/device.hpp"
#include "terralio/types.hpp"

namespace terralio::terrain {

struct TerrainObservation {
  std::vector<Vec2> xy;
  std::vector<double> z;

  std::size_t size() const { return xy.size(); }
  // center_select.cpp:9-16 (the device repeats this check before any state
  // change; here it is the reference's standalone call)
  void validate() const {
    if (xy.size() != z.size()) throw std::invalid_argument("observation xy/z length mismatch");
    if (xy.empty()) throw std::invalid_argument("empty observation");
    for (std::size_t i = 0; i < xy.size(); ++i)
      if (!std::isfinite(xy[i].x()) || !std::isfinite(xy[i].y()) || !std::isfinite(z[i]))
        throw std::invalid_argument("non-finite observation coordinate");
  }
};

struct CenterSet {
  std::vector<Vec2> centers;
  double mesh_resolution = 0.07;
  double accept_radius = 0.07;
  int accept_count = 3;
  Rect roi;

  tlg_center_params c_params() const {
    return {mesh_resolution, accept_radius, accept_count, 0,
            roi.min.x(),     roi.min.y(),   roi.max.x(), roi.max.y()};
  }
};

namespace detail {
// SoA host copies of a Vec2 list (the C-ABI takes x[], y[])
struct XY {
  std::vector<double> x, y;
  explicit XY(const std::vector<Vec2>& v) : x(v.size()), y(v.size()) {
    for (std::size_t i = 0; i < v.size(); ++i) {
      x[i] = v[i].x();
      y[i] = v[i].y();
    }
  }
};
using NodeFn = tlg_status (*)(tlg_ctx*, const double*, const double*, const double*, size_t, size_t,
                              tlg_mem, const tlg_center_params*, double*, double*, size_t, size_t*,
                              tlg_mem);
inline std::vector<Vec2> nodes(NodeFn fn, const TerrainObservation& obs, const tlg_center_params& cp) {
  const XY s(obs.xy);
  size_t cap = std::max<size_t>(64, obs.xy.size()), n = 0;
  std::vector<double> ox(cap), oy(cap);
  auto call = [&] {
    return fn(::terralio::detail::Device::ctx(), s.x.data(), s.y.data(), obs.z.data(), obs.xy.size(),
              obs.z.size(), TLG_HOST, &cp, ox.data(), oy.data(), cap, &n, TLG_HOST);
  };
  tlg_status st = call();
  if (st == TLG_BUFFER_TOO_SMALL) {
    cap = n;
    ox.resize(cap);
    oy.resize(cap);
    st = call();
  }
  ::terralio::detail::tlg_check(st);
  std::vector<Vec2> out(n);
  for (size_t i = 0; i < n; ++i) out[i] = Vec2(ox[i], oy[i]);
  return out;
}
}  // namespace detail

inline std::vector<Vec2> supported_mesh_nodes(const TerrainObservation& points, const Rect& roi,
                                              double mesh_resolution, double accept_radius,
                                              int accept_count) {
  CenterSet p;
  p.roi = roi;
  p.mesh_resolution = mesh_resolution;
  p.accept_radius = accept_radius;
  p.accept_count = accept_count;
  return detail::nodes(&tlg_supported_mesh_nodes, points, p.c_params());
}

inline CenterSet select_centers(const TerrainObservation& points, const Rect& roi, double mesh_resolution,
                                double accept_radius, int accept_count) {
  CenterSet set;
  set.roi = roi;
  set.mesh_resolution = mesh_resolution;
  set.accept_radius = accept_radius;
  set.accept_count = accept_count;
  set.centers = detail::nodes(&tlg_select_centers, points, set.c_params());
  return set;
}

}  // namespace terralio::terrain
