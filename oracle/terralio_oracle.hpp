// TEST INFRASTRUCTURE — CPU oracle for the terralio RBF terrain hot path.
//
// This is a plain-C++ restatement (no Eigen) of the reference CPU library
// under /root/reference/proj/core, written so the GPU product path can be
// checked against it. It is NOT part of the product: only tests/, the
// smoke() check in __graft_entry__.py and bench.py's cpu_baseline /
// --impl reference legs may load it.
//
// Parity pin: the reference cannot be compiled here (Eigen3 and the
// vendored doctest are absent), so this restatement is
// pinned against the reference's own hot-path unit tests and acceptance
// criteria, re-expressed in tests/test_oracle_*.py (closed forms, brute-force
// neighbour counts, dense ridge / dense inverse oracles, FD checks).
//
// Arithmetic contract: built -O3 -ffp-contract=off with no -march (x86-64
// SSE2 doubles, glibc exp), i.e. the reference's own Release flags
// (proj/CMakeLists.txt), so every expression rounds like the reference's.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace oracle {

struct V2 {
  double x = 0.0, y = 0.0;
};
struct V3 {
  double x = 0.0, y = 0.0, z = 0.0;
};
// Row-major 3x3.
struct M3 {
  double a[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  double operator()(int r, int c) const { return a[3 * r + c]; }
  double& operator()(int r, int c) { return a[3 * r + c]; }
};

// Column-major dense matrix (Eigen::MatrixXd default storage order).
struct Mat {
  long rows = 0, cols = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(long r, long c) : rows(r), cols(c), a(static_cast<size_t>(r * c), 0.0) {}
  double& operator()(long r, long c) { return a[static_cast<size_t>(c * rows + r)]; }
  double operator()(long r, long c) const { return a[static_cast<size_t>(c * rows + r)]; }
};

// --- types.hpp:14-25 -------------------------------------------------------
struct Rect {
  V2 min, max;
  bool contains(const V2& p) const {
    return p.x >= min.x && p.x <= max.x && p.y >= min.y && p.y <= max.y;
  }
  Rect dilated(double m) const { return {{min.x - m, min.y - m}, {max.x + m, max.y + m}}; }
};

inline double sqnorm(double dx, double dy) { return dx * dx + dy * dy; }

// --- grid_index.hpp:16-66 --------------------------------------------------
class GridIndex2 {
 public:
  explicit GridIndex2(double cell) : cell_(cell) {}
  std::uint32_t insert(const V2& p);
  void build(const std::vector<V2>& pts);
  std::vector<std::uint32_t> radius_query(const V2& q, double radius) const;
  std::size_t size() const { return points_.size(); }

 private:
  int coord(double v) const;
  static std::int64_t pack(int x, int y) {
    return (static_cast<std::int64_t>(x) << 32) ^
           static_cast<std::int64_t>(static_cast<std::uint32_t>(y));
  }
  double cell_;
  std::unordered_map<std::int64_t, std::vector<std::uint32_t>> cells_;
  std::vector<V2> points_;
};

// --- kernel.hpp / kernel.cpp ------------------------------------------------
struct KernelParams {
  double sigma = 0.04;
  double sigma_eps = 0.1;
  double lambda = 1e-3;
  double cutoff_radius = 0.0;
  double sigma_tilde() const;
  double moment_scale() const;
  void finalize();
};

double kernel_eval(const KernelParams& p, const V2& x, const V2& c, double bandwidth);

struct SparseVec {
  std::vector<std::pair<std::uint32_t, double>> entries;
};

// --- center_select.hpp / .cpp ----------------------------------------------
struct TerrainObservation {
  std::vector<V2> xy;
  std::vector<double> z;
  std::size_t size() const { return xy.size(); }
  void validate() const;
};

struct CenterSet {
  std::vector<V2> centers;
  double mesh_resolution = 0.07;
  double accept_radius = 0.07;
  int accept_count = 3;
  Rect roi;
};

struct NoSupportedCenters : std::runtime_error {
  NoSupportedCenters() : std::runtime_error("no supported centers") {}
};

std::vector<V2> supported_mesh_nodes(const TerrainObservation& pts, const Rect& roi,
                                     double res, double r_a, int count);
CenterSet select_centers(const TerrainObservation& pts, const Rect& roi, double res,
                         double r_a, int count);

// --- terrain_model.hpp / .cpp ----------------------------------------------
struct HeightQuery {
  double z = 0.0;
  bool supported = false;
};

struct UpdateReport {
  std::size_t active_blocks = 0, active_centers = 0, born_centers = 0;
  bool rejected = false;
};

class TerrainModel {
 public:
  TerrainModel() = default;
  TerrainModel(KernelParams kernel, CenterSet centers);
  TerrainModel(TerrainModel&&) = default;
  TerrainModel& operator=(TerrainModel&&) = default;

  const KernelParams& kernel() const { return kernel_; }
  const CenterSet& centers() const { return centers_; }
  const std::vector<double>& weights() const { return weights_; }
  std::size_t num_centers() const { return centers_.centers.size(); }
  std::size_t num_blocks() const { return blocks_.size(); }
  std::uint32_t block_of(std::uint32_t c) const { return block_index_[c]; }
  const std::vector<std::uint32_t>& block_members(std::uint32_t b) const {
    return blocks_[b].members;
  }
  const Mat& block_info_inverse(std::uint32_t b) const { return blocks_[b].info_inv; }

  SparseVec moment_feature(const V2& x) const;
  HeightQuery predict_height(const V2& x) const;
  V2 predict_gradient(const V2& x) const;
  UpdateReport recursive_update(const TerrainObservation& obs, bool allow_birth = true);
  std::vector<std::uint32_t> centers_near(const V2& x, double radius) const;

  void save(const std::string& path) const;
  static TerrainModel load(const std::string& path);

  // bench/test helper: overwrite the weight vector (size must match)
  void set_weights(const std::vector<double>& w) { weights_ = w; }

  friend TerrainModel fit_batch_ridge(const KernelParams&, const CenterSet&,
                                      const TerrainObservation&);

 private:
  struct Block {
    std::vector<std::uint32_t> members;
    Mat info_inv;
  };
  std::int64_t tile_key(const V2& c) const;
  std::uint32_t block_for_tile(std::int64_t key);
  std::uint32_t add_center(const V2& c);
  void rebuild_indexes();

  KernelParams kernel_;
  CenterSet centers_;
  std::vector<double> weights_;
  std::vector<std::uint32_t> block_index_;
  std::vector<Block> blocks_;
  std::unordered_map<std::int64_t, std::uint32_t> tile_blocks_;
  std::unique_ptr<GridIndex2> center_index_;
  std::unordered_map<std::int64_t, std::uint32_t> mesh_occupancy_;
};

TerrainModel fit_batch_ridge(const KernelParams& params, const CenterSet& centers,
                             const TerrainObservation& obs);

// --- so3.cpp:8-27 ----------------------------------------------------------
M3 hat(const V3& v);
M3 so3_exp(const V3& w);
M3 mul(const M3& a, const M3& b);
V3 mul(const M3& a, const V3& v);

// --- Manifold rows: contact.cpp:7-39 + scan_matcher.cpp:221-248 ------------
// Batched generalisation of the two wheel rows: row i uses lever arm h_i
// (sensor/base frame), xi_i = R h_i + t, r_i = xi_z - r_w - f(xi_xy).
struct ManifoldRow {
  double r = 0.0;      // scaled residual sqrt(lambda_M) * w_H * r_raw (0 when invalid)
  double J[6] = {0, 0, 0, 0, 0, 0};
  double raw = 0.0;    // unscaled residual (manifold_left/right analogue)
  bool valid = false;
};

ManifoldRow manifold_row(const TerrainModel& terrain, const M3& R, const V3& t, const V3& h,
                         double wheel_radius, double lambda_M, double huber_delta);

// Normal equations of stacked rows, scan_matcher.cpp:296-299 (A = J^T J,
// g = J^T r), accumulated in row order; plus cost = sum r^2 (:253).
struct NormalEq {
  double A[36] = {0};
  double g[6] = {0};
  double cost = 0.0;
  std::size_t valid = 0;
};
void accumulate(NormalEq& ne, const ManifoldRow& row);

// LM damped step, scan_matcher.cpp:300-305: delta = -(A + mu*diag(A)^+ +
// 1e-3 I)^-1 g via LDLT. Returns false when the solve is non-finite.
bool lm_step(const NormalEq& ne, double mu, double delta[6]);

// Pivoted LDL^T (Eigen::LDLT analogue: diagonal pivoting, "robust
// Cholesky"). Used by recursive_update (:221), fit_batch_ridge (:287,:304)
// and the LM step (:305).
struct Ldlt {
  long n = 0;
  Mat lu;                       // unit-lower L below diagonal, D on diagonal
  std::vector<long> perm;       // transpositions
  bool ok = true;               // no NaN pivot
  bool positive = true;         // all D >= 0
  explicit Ldlt(const Mat& a);
  Mat solve(const Mat& b) const;
  std::vector<double> solve(const std::vector<double>& b) const;
  std::vector<double> vectorD() const;
};

// --- Batch-predict consumers ----------------------------
// pipeline.cpp:150-170 select_ground_points: ground-labelled points (kind 2)
// in scan order, p = R f + t, kept when inside the ROI (types.hpp:18-21),
// within `radius` of the base in xy, and first in their xy voxel key
// (floor(x/voxel) << 21) ^ (floor(y/voxel) & (2^21 - 1)); stops after
// max_points kept. Returns the kept world points.
struct GroundPoints {
  std::vector<V2> xy;
  std::vector<double> z;
};
GroundPoints select_ground_points(const std::vector<V3>& p, const std::vector<std::uint8_t>& kind,
                                  const M3& R, const V3& t, const Rect& roi, double radius,
                                  double voxel, std::size_t max_points);

// metrics.cpp:199-232 terrain_error_histogram (kRange = 0.25 m).
struct Histogram {
  std::vector<double> edges;
  std::vector<std::size_t> counts;
  std::size_t trimmed = 0;
  std::size_t overflow = 0;
};
Histogram terrain_error_histogram(const TerrainModel& model, const std::vector<V2>& xy,
                                  const std::vector<double>& z, double trim_fraction, int bins);

// terrain_model.cpp:255-267 export_csv, numbers only: the supported grid
// points (x outer, y inner, both accumulated by += grid_step) and heights.
void export_grid(const TerrainModel& model, double grid_step, std::vector<double>& x,
                 std::vector<double>& y, std::vector<double>& z);


// --- Feature correspondences ------------------------------
// local_map.cpp:8-62 (sliding window of frames, per-frame voxel dedupe,
// ground hits kept as planar), kdtree.hpp:13-101 (exact k nearest within a
// gate, closest first, ties by smaller id — restated as an exhaustive search
// with the same ordering), scan_matcher.cpp:44-183 (build_correspondences),
// residuals.cpp:7-25 and scan_matcher.cpp:185-216 (feature rows of
// total_cost). Eigen's SelfAdjointEigenSolver is replaced by cyclic Jacobi
// (eigenvalues ascending, eigenvectors to ~1e-15): parity unpinned there.
struct MapConfig {
  double voxel_size = 0.1;
  std::size_t window = 20;
};
struct FeatureInput {  // one scan: sensor-frame points, kinds (0 edge, 1 planar, 2 ground), labels
  std::vector<V3> p;
  std::vector<std::uint8_t> kind;
  std::vector<std::int32_t> label;
};
// kdtree.hpp:13-101 restated (static median-split 3-d tree, same search and
// tie rules); knn() above is its exhaustive cross-check
class KdTree3 {
 public:
  void build(const std::vector<V3>& pts);
  std::vector<std::uint32_t> knn(const V3& q, int k, double gate) const;

 private:
  struct Node {
    std::uint32_t id;
    int left = -1, right = -1;
    int axis = 0;
  };
  int build_range(int b, int e, int depth);
  void search(int ni, const V3& q, int k, double gate2,
              std::vector<std::pair<double, std::uint32_t>>& heap) const;
  std::vector<V3> pts_;
  std::vector<std::uint32_t> order_;
  std::vector<Node> nodes_;
  int root_ = -1;
};

class LocalMap {
 public:
  explicit LocalMap(MapConfig c = {}) : cfg_(c) {}
  void insert(const FeatureInput& scan, const M3& R, const V3& t);
  std::vector<V3> edge, planar;
  std::vector<std::int32_t> edge_label, planar_label;
  KdTree3 edge_tree, planar_tree;
  bool use_tree = true;  // false: exhaustive kNN (cross-check)

 private:
  struct Frame {
    std::vector<V3> edge, planar;
    std::vector<std::int32_t> edge_label, planar_label;
  };
  MapConfig cfg_;
  std::vector<Frame> frames_;
};
std::vector<std::uint32_t> knn(const std::vector<V3>& pts, const V3& q, int k, double gate);
void eigen_sym3(const double A[9], double evals[3], double evecs[9]);  // evecs column-major

struct SolverConfigM {
  double corr_gate = 1.0, huber_delta = 0.1, plane_fit_tol = 0.025, plane_eig_ratio = 5.0;
  double edge_eig_ratio = 3.0, edge_fit_tol = 0.05, edge_min_extent = 0.05;
  double trim_ratio = 5.0, trim_floor = 0.003, ground_corr_voxel = 0.25, ground_corr_radius = 4.0;
};
struct Correspondence {
  int kind = 0;             // 0 edge, 1 planar
  std::uint32_t feature = 0;  // index into the scan
  V3 p_sensor, line_point, line_dir{1.0, 0.0, 0.0}, normal{0.0, 0.0, 1.0};
  double offset = 0.0, weight = 1.0;
  std::int32_t label = -1;
  double dist = 0.0, fitq = 0.0;
};
std::vector<Correspondence> build_correspondences(const FeatureInput& f, const M3& R, const V3& t,
                                                  const LocalMap& map, const SolverConfigM& cfg);
// feature rows of total_cost at pose (R, t), accumulated into ne in row order
void feature_normal_eq(const std::vector<Correspondence>& c, const M3& R, const V3& t,
                       NormalEq& ne, std::size_t* rows);

}  // namespace oracle
