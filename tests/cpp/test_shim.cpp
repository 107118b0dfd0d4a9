// C++ drop-in check: the reference's hot-path unit tests written against the
// C++ shim (include/terralio_b200/terrain.hpp), i.e. the way proj/core code
// calls the terrain model. Exit code = number of failed checks.
// Build: g++ -std=c++20 -Iinclude tests/cpp/test_shim.cpp -Lpaper_2509_26222_b200/lib
//        -lterralio_gpu -Wl,-rpath,...
#include <cmath>
#include <cstdio>
#include <random>

#include <cuda_runtime.h>

#include "terralio_b200/terrain.hpp"

using namespace terralio;
using namespace terralio::terrain;

static int failures = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #c);     \
      ++failures;                                                  \
    }                                                              \
  } while (0)

int main() {
  // kernel.cpp finalize (test_kernel.cpp:50-69)
  KernelParams k;
  k.finalize();
  CHECK(std::fabs(k.cutoff_radius - 3.0 * k.sigma_tilde()) < 1e-15);
  bool threw = false;
  try {
    KernelParams bad;
    bad.sigma = 0.0;
    bad.finalize();
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);

  // select_centers support rule (test_center_select.cpp:21-36)
  std::mt19937_64 rng(11);
  std::uniform_real_distribution<double> u(0.0, 2.0);
  TerrainObservation obs;
  for (int i = 0; i < 400; ++i) {
    obs.xy.push_back({u(rng), u(rng)});
    obs.z.push_back(0.1 * std::sin(4.0 * obs.xy.back().x()));
  }
  const Rect roi{{0.0, 0.0}, {2.0, 2.0}};
  const CenterSet set = select_centers(obs, roi, 0.1, 0.12, 3);
  CHECK(!set.centers.empty());
  for (const Vec2& c : set.centers) {
    int n = 0;
    for (const Vec2& p : obs.xy)
      n += std::hypot(p.x() - c.x(), p.y() - c.y()) <= 0.12;
    CHECK(roi.contains(c) && n >= 3);
  }
  threw = false;
  try {
    TerrainObservation far;
    far.xy.push_back({10.0, 10.0});
    far.z.push_back(0.0);
    select_centers(far, {{0.0, 0.0}, {1.0, 1.0}}, 0.1, 0.1, 3);
  } catch (const NoSupportedCenters&) {
    threw = true;
  }
  CHECK(threw);

  // model: recursive updates reproduce the batch fit (test_terrain_model.cpp:109-126)
  KernelParams kk;
  kk.sigma = 0.08;
  kk.sigma_eps = 0.05;
  kk.cutoff_radius = 10.0;
  kk.finalize();
  TerrainModel rec(kk, set);
  for (int s = 0; s < 4; ++s) {
    TerrainObservation part;
    part.xy.assign(obs.xy.begin() + s * 100, obs.xy.begin() + (s + 1) * 100);
    part.z.assign(obs.z.begin() + s * 100, obs.z.begin() + (s + 1) * 100);
    const UpdateReport r = rec.recursive_update(part, false);
    CHECK(!r.rejected);
  }
  const TerrainModel batch = fit_batch_ridge(kk, set, obs);
  const auto wr = rec.weights(), wb = batch.weights();
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < wr.size(); ++i) {
    num += (wr[i] - wb[i]) * (wr[i] - wb[i]);
    den += wb[i] * wb[i];
  }
  CHECK(std::sqrt(num / den) < 1e-8);

  // point-sharded batch ridge: two shards summed (host-side here) == one call
  {
    TerrainModel sh(kk, set);
    const TerrainModel::BatchSystem bs = sh.batch_system();
    double *H0, *H1, *b0, *b1;
    CHECK(cudaMalloc(&H0, bs.elems * 8) == cudaSuccess && cudaMalloc(&H1, bs.elems * 8) == cudaSuccess);
    CHECK(cudaMalloc(&b0, bs.n * 8) == cudaSuccess && cudaMalloc(&b1, bs.n * 8) == cudaSuccess);
    TerrainObservation s0, s1;
    s0.xy.assign(obs.xy.begin(), obs.xy.begin() + 150);
    s0.z.assign(obs.z.begin(), obs.z.begin() + 150);
    s1.xy.assign(obs.xy.begin() + 150, obs.xy.end());
    s1.z.assign(obs.z.begin() + 150, obs.z.end());
    sh.batch_assemble(s1, H1, b1, false);
    auto add_other = [&](double* dst, std::size_t count) {  // a two-rank "all-reduce"
      std::vector<double> a(count), c(count);
      cudaMemcpy(a.data(), dst, count * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(c.data(), dst == H0 ? H1 : b1, count * 8, cudaMemcpyDeviceToHost);
      for (std::size_t i = 0; i < count; ++i) a[i] += c[i];
      cudaMemcpy(dst, a.data(), count * 8, cudaMemcpyHostToDevice);
    };
    fit_batch_ridge_sharded(sh, s0, true, H0, b0, add_other);
    const auto ws = sh.weights();
    double n2 = 0.0, d2 = 0.0;
    for (std::size_t i = 0; i < ws.size(); ++i) {
      n2 += (ws[i] - wb[i]) * (ws[i] - wb[i]);
      d2 += wb[i] * wb[i];
    }
    CHECK(std::sqrt(n2 / d2) < 1e-10);
    cudaFree(H0);
    cudaFree(H1);
    cudaFree(b0);
    cudaFree(b1);
  }

  // the library's own communicator (tlg_comm, one rank here): the sharded fit
  // of the whole set equals the single call
  {
    TerrainModel sh(kk, set);
    const Communicator comm(Communicator::unique_id(), 0, 1);
    fit_batch_ridge_sharded(sh, comm, obs);
    const auto ws = sh.weights();
    bool same = ws.size() == wb.size();
    for (std::size_t i = 0; same && i < ws.size(); ++i) same = ws[i] == wb[i];
    CHECK(same);
  }

  // predict_height / unsupported (test_terrain_model.cpp:79-100)
  const HeightQuery q = batch.predict_height({1.0, 1.0});
  CHECK(q.supported);
  const HeightQuery far = batch.predict_height({50.0, 50.0});
  CHECK(!far.supported && far.z == 0.0);
  threw = false;
  try {
    batch.predict_height({NAN, 0.0});
  } catch (const std::domain_error&) {
    threw = true;
  }
  CHECK(threw);

  // snapshot round trip (test_terrain_model.cpp:226-241)
  batch.save("/tmp/terralio_b200_shim.bin");
  const TerrainModel loaded = TerrainModel::load("/tmp/terralio_b200_shim.bin");
  CHECK(loaded.num_centers() == batch.num_centers());
  CHECK(std::fabs(loaded.predict_height({1.0, 1.0}).z - q.z) <= 1e-14 * std::fabs(q.z) + 1e-300);

  // metrics.cpp:199-232 through the shim: counts add up, edges as the reference's
  {
    std::vector<Vec2> qs;
    std::vector<double> zs;
    for (int i = 0; i < 2000; ++i) {
      qs.push_back({u(rng), u(rng)});
      zs.push_back(0.1 * std::sin(4.0 * qs.back().x()));
    }
    const eval::Histogram h = eval::terrain_error_histogram(batch, qs, zs, 0.1, 25);
    CHECK(h.trimmed == 200);
    CHECK(h.total() == 1800);
    CHECK(h.edges.size() == 26 && h.edges[25] == 0.25);
    batch.export_csv("/tmp/terralio_b200_shim.csv", 0.05);
  }

  // match: map, correspondences, feature normal equations, LM step
  {
    match::LocalMap lmap;
    match::FeatureCloud cloud;
    std::uniform_real_distribution<double> uu(-2.0, 2.0);
    for (int i = 0; i < 6000; ++i) {
      match::FeaturePoint f;
      if (i % 3 == 0)
        f = {{uu(rng), uu(rng), 0.0}, match::FeatureKind::Ground, 0};
      else if (i % 3 == 1)
        f = {{2.5, uu(rng), 1.0 + 0.5 * uu(rng)}, match::FeatureKind::Planar, 1};
      else
        f = {{uu(rng), 2.5, 1.0 + 0.5 * uu(rng)}, match::FeatureKind::Planar, 2};
      cloud.points.push_back(f);
    }
    lmap.insert(cloud, Mat3::Identity(), Vec3{0.0, 0.0, 0.0});
    CHECK(!lmap.empty());
    match::SolverConfig sc;
    const auto corr = match::build_correspondences(cloud, Mat3::Identity(), Vec3{0.01, 0.0, 0.0},
                                                   lmap, sc);
    CHECK(corr.size() > 100);
    const tlg_normal_eq fne = match::feature_normal_eq(lmap, Mat3::Identity(), Vec3{0.01, 0.0, 0.0});
    CHECK(fne.valid == static_cast<double>(corr.size()));
    double delta[6];
    CHECK(match::lm_step(fne, 1e-4, delta));
  }

  // manifold rows + normal equations
  std::vector<Vec3> lever;
  for (int i = 0; i < 1000; ++i) lever.push_back({u(rng), u(rng), 0.05});
  const auto rows = kin::manifold_rows(batch, Mat3::Identity(), Vec3{0.0, 0.0, 0.0}, lever, 0.0,
                                       1.0, 0.05);
  CHECK(rows.ne.valid > 900);
  CHECK(rows.ne.cost > 0.0);
  std::printf("test_shim: %d failure(s)\n", failures);
  return failures;
}
