// terralio drop-in: proj/core/include/terralio/kinematics/contact.hpp:9-24.
// The wheel's lever arm h = chain_end_position(q) (host FK) feeds the device
// manifold row (tlg_manifold_rows, one row, lambda_M = 1, no Huber): the
// residual xi_z - r_w - f(xi_xy) with xi = R h + t, and its 1x6 Jacobian
// [-df/dx, -df/dy, 1] [-R hat(h), I] (contact.cpp:7-39).
#pragma once

#include <Eigen/Core>

#include "terralio/detail/device.hpp"
#include "terralio/kinematics/leg_model.hpp"
#include "terralio/so3.hpp"
#include "terralio/terrain/terrain_model.hpp"

namespace terralio::kin {

struct ManifoldResidual {
  double value = 0.0;
  bool valid = false;
  Vec3 wheel_center = Vec3::Zero();
};

namespace detail {
inline Vec3 lever_arm(const JointConfig& joints, const LegModel& leg, Side side) {
  const LegChain& chain = leg.chain(side);
  const std::span<const double> q(joints.angles.data() + leg.joint_offset(side),
                                  static_cast<std::size_t>(chain.joint_count()));
  return chain_end_position(chain, q);
}
struct Row {
  double raw = 0.0, J[6] = {0, 0, 0, 0, 0, 0};
  bool valid = false;
};
inline Row device_row(const RobotState& s, const Vec3& h, double wheel_radius, const terrain::TerrainModel& t) {
  double R[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R[3 * i + j] = s.rotation(i, j);
  const double tv[3] = {s.translation.x(), s.translation.y(), s.translation.z()};
  const double hx = h.x(), hy = h.y(), hz = h.z();
  Row row;
  double r = 0.0;
  uint8_t v = 0;
  if (t.handle())
    ::terralio::detail::tlg_check(tlg_manifold_rows(t.handle(), R, tv, &hx, &hy, &hz, 1, TLG_HOST, wheel_radius, 1.0,
                                                    0.0, &r, row.J, &v, &row.raw, TLG_HOST, nullptr));
  row.valid = v != 0;
  return row;
}
}  // namespace detail

inline ManifoldResidual manifold_residual(const RobotState& state, const JointConfig& joints, const LegModel& leg,
                                          Side side, const terrain::TerrainModel& terrain) {
  ManifoldResidual out;
  out.wheel_center = wheel_center_world(state, joints, leg, side);
  const detail::Row row = detail::device_row(state, detail::lever_arm(joints, leg, side), leg.wheel_radius, terrain);
  if (!row.valid) return out;
  out.valid = true;
  out.value = row.raw;
  return out;
}

inline Eigen::Matrix<double, 1, 6> manifold_jacobian(const RobotState& state, const JointConfig& joints,
                                                     const LegModel& leg, Side side,
                                                     const terrain::TerrainModel& terrain) {
  const Vec3 h = detail::lever_arm(joints, leg, side);
  const detail::Row row = detail::device_row(state, h, leg.wheel_radius, terrain);
  Eigen::Matrix<double, 1, 6> J;
  if (row.valid) {
    for (int c = 0; c < 6; ++c) J(0, c) = row.J[c];
    return J;
  }
  // no centre in reach: the reference's gradient is zero there, leaving
  // d(xi_z)/d[dtheta, dt] = the z row of [-R hat(h), I]
  const Mat3 Rh = state.rotation * hat(h);
  J << -Rh(2, 0), -Rh(2, 1), -Rh(2, 2), 0.0, 0.0, 1.0;
  return J;
}

}  // namespace terralio::kin
