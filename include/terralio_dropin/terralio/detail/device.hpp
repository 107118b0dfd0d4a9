// terralio drop-in (Eigen-typed) — device plumbing shared by the drop-in
// headers: the process-wide tlg_ctx and the status -> exception mapping of
// the reference (std::invalid_argument, std::domain_error,
// NoSupportedCenters, std::runtime_error).
//
// These headers replace proj/core/include/terralio/{types,so3}.hpp,
// terrain/{kernel,center_select,terrain_model}.hpp and
// kinematics/{leg_model,contact}.hpp with the same names, signatures and
// Eigen types; every data-sized computation runs through the C-ABI
// (include/terralio_gpu.h) on the GPU. Put include/terralio_dropin first on
// the include path of code written against the reference.
#pragma once

#include <new>
#include <stdexcept>
#include <string>

#include "../../../terralio_gpu.h"

namespace terralio {
namespace terrain {
// center_select.hpp:30-32
struct NoSupportedCenters : std::runtime_error {
  NoSupportedCenters() : std::runtime_error("no supported centers") {}
};
}  // namespace terrain
namespace detail {

[[noreturn]] inline void throw_tlg(tlg_status st) {
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

inline void tlg_check(tlg_status st) {
  if (st != TLG_OK) throw_tlg(st);
}

// Device 0, the legacy default stream (tlg_ctx_create with NULL).
class Device {
 public:
  static tlg_ctx* ctx() {
    static Device d;
    return d.ctx_;
  }
  ~Device() { tlg_ctx_destroy(ctx_); }

 private:
  Device() { tlg_check(tlg_ctx_create(0, nullptr, &ctx_)); }
  tlg_ctx* ctx_ = nullptr;
};

}  // namespace detail
}  // namespace terralio
