// terralio drop-in: proj/core/include/terralio/terrain/kernel.hpp:12-34.
// finalize runs the C-ABI's tlg_kernel_finalize; kernel_eval one pair on the
// device (tlg_kernel_eval; batch callers pass arrays to the C-ABI directly).
#pragma once

#include <cmath>
#include <cstdint>
#include <utility>
#include <vector>

#include "terralio/detail/device.hpp"
#include "terralio/types.hpp"

namespace terralio::terrain {

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
    tlg_kernel_params p = c_params();
    ::terralio::detail::tlg_check(tlg_kernel_finalize(&p));
    cutoff_radius = p.cutoff_radius;
  }
  tlg_kernel_params c_params() const { return {sigma, sigma_eps, lambda, cutoff_radius}; }
};

inline double kernel_eval(const KernelParams& params, const Vec2& x, const Vec2& c, double bandwidth) {
  const tlg_kernel_params p = params.c_params();
  const double xs[2] = {x.x(), x.y()}, cs[2] = {c.x(), c.y()};
  double out = 0.0;
  ::terralio::detail::tlg_check(tlg_kernel_eval(::terralio::detail::Device::ctx(), &p, &xs[0], &xs[1], &cs[0], &cs[1], 1,
                                    TLG_HOST, bandwidth, &out, TLG_HOST));
  return out;
}

struct SparseVec {
  std::vector<std::pair<std::uint32_t, double>> entries;
};

}  // namespace terralio::terrain
