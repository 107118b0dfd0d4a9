// terralio drop-in: proj/core/include/terralio/match/scan_matcher.hpp:15-105
// (scan_matcher.cpp:44-358 semantics) on the device: association
// (tlg_build_correspondences, the exact kNN of the reference's kd-tree and
// its gates/trims), total_cost's rows (tlg_feature_rows + the wheel
// manifold rows, tlg_manifold_rows) and lm_solve, whose O(1) control flow
// (the damping schedule, acceptance, convergence tests and the SE(3)
// retraction) stays on the host while every data-sized step runs on the GPU:
// the correspondences stay in the map object across the inner iterations and
// each cost evaluation is one reduction to the 6x6 normal equations.
#pragma once

#include <Eigen/Core>
#include <cmath>
#include <optional>
#include <stdexcept>
#include <vector>

#include "terralio/detail/device.hpp"
#include "terralio/kinematics/contact.hpp"
#include "terralio/match/local_map.hpp"
#include "terralio/match/residuals.hpp"
#include "terralio/so3.hpp"
#include "terralio/terrain/terrain_model.hpp"
#include "terralio/types.hpp"

namespace terralio::match {

struct SolverConfig {
  double lambda_manifold = 1.0;
  double lm_init_damping = 1e-4;
  int lm_max_iters = 10;
  int lm_max_inner = 8;
  int lm_max_rejects = 12;
  double tol_dcost = 1e-10;
  double tol_dstate = 1e-10;
  double corr_gate = 1.0;
  int min_correspondences = 10;
  double huber_delta = 0.1;
  double manifold_huber_delta = 0.05;
  double plane_fit_tol = 0.025;
  double plane_eig_ratio = 5.0;
  double edge_eig_ratio = 3.0;
  double edge_fit_tol = 0.05;
  double edge_min_extent = 0.05;
  double degeneracy_eig_min = 10.0;
  double trim_ratio = 5.0;
  double trim_floor = 0.003;
  double ground_corr_voxel = 0.25;
  double ground_corr_radius = 4.0;

  tlg_match_config c_config() const {
    return {corr_gate,    huber_delta,     plane_fit_tol, plane_eig_ratio, edge_eig_ratio, edge_fit_tol,
            edge_min_extent, trim_ratio, trim_floor,    ground_corr_voxel, ground_corr_radius};
  }
};

struct Correspondence {
  FeatureKind kind = FeatureKind::Edge;
  Vec3 p_sensor = Vec3::Zero();
  LineParam line;
  PlaneParam plane;
  double weight = 1.0;
  std::int32_t map_label = -1;
};

struct ManifoldInputs {
  const JointConfig* joints = nullptr;
  const kin::LegModel* leg = nullptr;
  const terrain::TerrainModel* terrain = nullptr;
  bool enabled() const { return joints && leg && terrain; }
};

struct CostEval {
  double cost = 0.0;
  Eigen::MatrixXd jacobian;  // rows x 6, columns [dtheta, dt]
  Eigen::VectorXd residual;
  int feature_rows = 0;
  int manifold_rows = 0;
  std::optional<double> manifold_left, manifold_right;
};

struct SolveReport {
  bool converged = false;
  bool failed = false;
  bool degenerate = false;
  int outer_iterations = 0;
  int accepted_steps = 0;
  double final_cost = 0.0;
  std::size_t correspondence_count = 0;
  std::vector<double> cost_trace;
  std::optional<double> manifold_left, manifold_right;
  double smallest_feature_eigenvalue = 0.0;
};

namespace detail {
struct Pose9 {
  double R[9], t[3];
  explicit Pose9(const RobotState& s) {
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) R[3 * i + j] = s.rotation(i, j);
    for (int i = 0; i < 3; ++i) t[i] = s.translation(i);
  }
};
struct Scan {
  std::vector<double> x, y, z;
  std::vector<uint8_t> kind;
  explicit Scan(const FeatureCloud& f) {
    for (const auto& p : f.points) {
      x.push_back(p.p.x());
      y.push_back(p.p.y());
      z.push_back(p.p.z());
      kind.push_back(static_cast<uint8_t>(p.kind));
    }
  }
};
// the two wheels' lever arms (base frame) and the terrain to evaluate on
struct Wheels {
  bool on = false;
  double hx[2], hy[2], hz[2], radius = 0.0;
  const terrain::TerrainModel* terrain = nullptr;
  Wheels(const ManifoldInputs& mi, const SolverConfig& cfg) {
    if (!(mi.enabled() && cfg.lambda_manifold > 0.0)) return;
    on = true;
    terrain = mi.terrain;
    radius = mi.leg->wheel_radius;
    int s = 0;
    for (const kin::Side side : {kin::Side::Left, kin::Side::Right}) {
      const Vec3 h = kin::detail::lever_arm(*mi.joints, *mi.leg, side);
      hx[s] = h.x();
      hy[s] = h.y();
      hz[s] = h.z();
      ++s;
    }
  }
  // the two rows (scan_matcher.cpp:221-248): weighted r / J, valid, raw
  void rows(const RobotState& st, const SolverConfig& cfg, double r[2], double J[12], uint8_t v[2],
            double raw[2], tlg_normal_eq* ne) const {
    const Pose9 P(st);
    ::terralio::detail::tlg_check(tlg_manifold_rows(terrain->handle(), P.R, P.t, hx, hy, hz, 2, TLG_HOST, radius,
                                                    cfg.lambda_manifold, cfg.manifold_huber_delta, r, J, v, raw,
                                                    TLG_HOST, ne));
  }
};
inline void add_ne(tlg_normal_eq& a, const tlg_normal_eq& b) {
  for (int k = 0; k < 21; ++k) a.A[k] += b.A[k];
  for (int k = 0; k < 6; ++k) a.g[k] += b.g[k];
  a.cost += b.cost;
  a.valid += b.valid;
}
}  // namespace detail

// scan_matcher.cpp:44-183 at the guess pose; the device keeps the result
// (lm_solve reuses it), this returns a host copy in the reference's types.
inline std::vector<Correspondence> build_correspondences(const FeatureCloud& features, const RobotState& guess,
                                                         const LocalMap& map, const SolverConfig& config) {
  std::vector<Correspondence> out;
  if (map.empty()) return out;
  const detail::Scan s(features);
  const detail::Pose9 P(guess);
  const tlg_match_config c = config.c_config();
  std::size_t n = 0;
  ::terralio::detail::tlg_check(tlg_build_correspondences(map.handle(), s.x.data(), s.y.data(), s.z.data(),
                                                          s.kind.data(), s.x.size(), TLG_HOST, P.R, P.t, &c, &n));
  std::vector<int32_t> kind(n), label(n);
  std::vector<uint32_t> feat(n);
  std::vector<double> par(7 * n), w(n);
  ::terralio::detail::tlg_check(tlg_correspondences_get(map.handle(), kind.data(), feat.data(), par.data(),
                                                        w.data(), label.data(), nullptr, nullptr, n));
  out.resize(n);
  for (std::size_t i = 0; i < n; ++i) {
    Correspondence& o = out[i];
    const double* p = &par[7 * i];
    o.kind = kind[i] == 0 ? FeatureKind::Edge : FeatureKind::Planar;
    o.p_sensor = features.points[feat[i]].p;
    if (kind[i] == 0) {
      o.line.point = Vec3(p[0], p[1], p[2]);
      o.line.direction = Vec3(p[3], p[4], p[5]);
    } else {
      o.plane.normal = Vec3(p[0], p[1], p[2]);
      o.plane.offset = p[3];
    }
    o.weight = w[i];
    o.map_label = label[i];
  }
  return out;
}

// scan_matcher.cpp:185-255: feature rows then the two wheel rows (zero rows
// when unsupported); throws std::runtime_error when nothing is left.
inline CostEval total_cost(const RobotState& state, const std::vector<Correspondence>& correspondences,
                           const ManifoldInputs& manifold, const SolverConfig& config) {
  const std::size_t nc = correspondences.size();
  std::vector<int32_t> kind(nc);
  std::vector<double> ps(3 * nc), par(7 * nc, 0.0), w(nc);
  std::size_t frows = 0;
  for (std::size_t i = 0; i < nc; ++i) {
    const Correspondence& c = correspondences[i];
    kind[i] = c.kind == FeatureKind::Edge ? 0 : 1;
    frows += kind[i] == 0 ? 3 : 1;
    for (int a = 0; a < 3; ++a) ps[3 * i + a] = c.p_sensor(a);
    if (kind[i] == 0) {
      for (int a = 0; a < 3; ++a) {
        par[7 * i + a] = c.line.point(a);
        par[7 * i + 3 + a] = c.line.direction(a);
      }
    } else {
      for (int a = 0; a < 3; ++a) par[7 * i + a] = c.plane.normal(a);
      par[7 * i + 3] = c.plane.offset;
    }
    w[i] = c.weight;
  }
  const detail::Wheels wheels(manifold, config);
  const Eigen::Index rows = static_cast<Eigen::Index>(frows) + (wheels.on ? 2 : 0);
  CostEval ev;
  ev.jacobian.resize(rows, 6);
  ev.residual.resize(rows);
  std::vector<double> fr(frows), fJ(6 * frows);
  std::size_t got = 0;
  const detail::Pose9 P(state);
  if (nc)
    ::terralio::detail::tlg_check(tlg_feature_rows(::terralio::detail::Device::ctx(), kind.data(), ps.data(),
                                                   par.data(), w.data(), nc, P.R, P.t, fr.data(), fJ.data(),
                                                   frows, &got));
  for (std::size_t r = 0; r < frows; ++r) {
    ev.residual(static_cast<Eigen::Index>(r)) = fr[r];
    for (int c = 0; c < 6; ++c) ev.jacobian(static_cast<Eigen::Index>(r), c) = fJ[r + c * frows];
  }
  ev.feature_rows = static_cast<int>(frows);
  if (wheels.on) {
    double r[2], J[12], raw[2];
    uint8_t v[2];
    wheels.rows(state, config, r, J, v, raw, nullptr);
    for (int s = 0; s < 2; ++s) {
      const Eigen::Index row = static_cast<Eigen::Index>(frows) + s;
      ev.residual(row) = r[s];
      for (int c = 0; c < 6; ++c) ev.jacobian(row, c) = J[s + 2 * c];
      if (v[s]) {
        (s == 0 ? ev.manifold_left : ev.manifold_right) = raw[s];
        ++ev.manifold_rows;
      }
    }
  }
  if (ev.residual.size() == 0 || (ev.feature_rows == 0 && ev.manifold_rows == 0))
    throw std::runtime_error("nothing to optimize");
  ev.cost = ev.residual.squaredNorm();
  return ev;
}

// scan_matcher.cpp:257-358. Each cost evaluation is the device reduction of
// the rows to A = J^T J, g = J^T r (tlg_feature_normal_eq over the map's
// correspondences + the wheel rows); the damped step is tlg_lm_step.
inline RobotState lm_solve(const RobotState& initial, const FeatureCloud& features, const LocalMap& map,
                           const ManifoldInputs& manifold, const SolverConfig& config,
                           SolveReport* report = nullptr) {
  SolveReport local;
  SolveReport& rep = report ? *report : local;
  rep = SolveReport{};
  tlg_ctx* ctx = ::terralio::detail::Device::ctx();
  const detail::Wheels wheels(manifold, config);
  const detail::Scan scan(features);
  const tlg_match_config mc = config.c_config();
  struct Eval {
    tlg_normal_eq ne{}, feat{};
    std::optional<double> left, right;
  };
  auto cost = [&](const RobotState& s) {
    Eval e;
    const detail::Pose9 P(s);
    ::terralio::detail::tlg_check(tlg_feature_normal_eq(map.handle(), P.R, P.t, &e.feat));
    e.ne = e.feat;
    if (wheels.on) {
      double r[2], J[12], raw[2];
      uint8_t v[2];
      tlg_normal_eq nm{};
      wheels.rows(s, config, r, J, v, raw, &nm);
      detail::add_ne(e.ne, nm);
      if (v[0]) e.left = raw[0];
      if (v[1]) e.right = raw[1];
    }
    if (e.ne.valid == 0) throw std::runtime_error("nothing to optimize");
    return e;
  };
  RobotState state = initial;
  double mu = config.lm_init_damping;
  int rejects = 0;
  for (int outer = 0; outer < config.lm_max_iters; ++outer) {
    ++rep.outer_iterations;
    std::size_t nc = 0;
    if (!map.empty()) {
      const detail::Pose9 P(state);
      ::terralio::detail::tlg_check(tlg_build_correspondences(map.handle(), scan.x.data(), scan.y.data(),
                                                              scan.z.data(), scan.kind.data(), scan.x.size(),
                                                              TLG_HOST, P.R, P.t, &mc, &nc));
    }
    rep.correspondence_count = nc;
    if (static_cast<int>(nc) < config.min_correspondences) {
      rep.degenerate = true;
      break;
    }
    Eval ev = cost(state);
    rep.cost_trace.push_back(ev.ne.cost);
    rep.final_cost = ev.ne.cost;
    rep.manifold_left = ev.left;
    rep.manifold_right = ev.right;
    double lam = 0.0;
    ::terralio::detail::tlg_check(tlg_ne_min_eigenvalue(ctx, &ev.feat, &lam));
    rep.smallest_feature_eigenvalue = lam;
    if (lam < config.degeneracy_eig_min) rep.degenerate = true;
    bool improved = false, local_converged = false;
    double moved = 0.0;
    for (int inner = 0; inner < config.lm_max_inner; ++inner) {
      double d[6];
      if (tlg_lm_step(ctx, &ev.ne, mu, d) != TLG_OK) {
        rep.failed = true;
        return initial;
      }
      const Vec3 dth(d[0], d[1], d[2]), dt(d[3], d[4], d[5]);
      const double dn = std::sqrt(dth.squaredNorm() + dt.squaredNorm());
      if (dn < config.tol_dstate) {
        local_converged = true;
        break;
      }
      RobotState cand = state;
      cand.rotation = state.rotation * so3_exp(dth);
      reorthonormalize(cand.rotation);
      cand.translation = state.translation + dt;
      Eval ce = cost(cand);
      if (ce.ne.cost < ev.ne.cost) {
        const double dcost = ev.ne.cost - ce.ne.cost;
        state = cand;
        ev = ce;
        rep.cost_trace.push_back(ev.ne.cost);
        rep.final_cost = ev.ne.cost;
        rep.manifold_left = ev.left;
        rep.manifold_right = ev.right;
        mu = std::max(mu * 0.1, 1e-12);
        ++rep.accepted_steps;
        improved = true;
        rejects = 0;
        moved += dn;
        if (dcost < config.tol_dcost || dn < config.tol_dstate) {
          local_converged = true;
          break;
        }
      } else {
        mu *= 10.0;
        if (++rejects > config.lm_max_rejects) {
          if (rep.accepted_steps == 0) {
            rep.failed = true;
            return initial;
          }
          local_converged = true;
          break;
        }
      }
    }
    if (local_converged && moved < 1e-9) {
      rep.converged = true;
      break;
    }
    if (!improved && !local_converged && rep.accepted_steps > 0) {
      rep.converged = true;
      break;
    }
    if (rep.degenerate && !improved) break;
  }
  return state;
}

}  // namespace terralio::match
