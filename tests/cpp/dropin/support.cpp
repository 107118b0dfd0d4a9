// TEST SUPPORT for the drop-in check: the reference's own unit-test files
// (proj/tests/unit/test_{kernel,center_select,terrain_model,kinematics}.cpp,
// compiled in place from /root/reference by paper_2509_26222_b200/build.py)
// are built against include/terralio_dropin (the Eigen-typed drop-in over the
// GPU C-ABI) and linked with libterralio_gpu.so. This file supplies the
// doctest runner (oracle/shims/doctest.h) and the one out-of-scope symbol
// those tests use: sim::default_robot, the two-leg robot of the stock
// scenes (scene.cpp:12-28), restated.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include "terralio/kinematics/leg_model.hpp"

namespace terralio::sim {

kin::LegModel default_robot() {
  kin::LegModel robot;
  robot.wheel_radius = 0.08;
  for (const kin::Side s : {kin::Side::Left, kin::Side::Right}) {
    const double y = (s == kin::Side::Left) ? 0.12 : -0.12;
    kin::LegChain& c = (s == kin::Side::Left) ? robot.left : robot.right;
    c.links = {{"hip", "base", Vec3(0.0, y, -0.08), Vec3::UnitY(), true},
               {"knee", "hip", Vec3(0.0, 0.0, -0.24), Vec3::UnitY(), true},
               {"wheel", "knee", Vec3(0.0, 0.0, -0.24), Vec3::UnitY(), false}};
  }
  return robot;
}

}  // namespace terralio::sim
