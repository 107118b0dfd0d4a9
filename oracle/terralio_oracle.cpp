// TEST INFRASTRUCTURE — CPU restatement of the reference hot path.
// See terralio_oracle.hpp for the contract. Each function cites the
// reference file:line (under /root/reference/proj/core) it follows.
#include "terralio_oracle.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <limits>
#include <map>
#include <set>
#include <unordered_set>

namespace oracle {

// ---------------------------------------------------------------------------
// grid_index.hpp:20-61
std::uint32_t GridIndex2::insert(const V2& p) {
  const auto id = static_cast<std::uint32_t>(points_.size());
  points_.push_back(p);
  cells_[pack(coord(p.x), coord(p.y))].push_back(id);
  return id;
}

void GridIndex2::build(const std::vector<V2>& pts) {
  points_.reserve(points_.size() + pts.size());
  for (const V2& p : pts) insert(p);
}

int GridIndex2::coord(double v) const { return static_cast<int>(std::floor(v / cell_)); }

std::vector<std::uint32_t> GridIndex2::radius_query(const V2& q, double radius) const {
  std::vector<std::uint32_t> out;
  const double r2 = radius * radius;
  const int span = static_cast<int>(std::ceil(radius / cell_));
  const int cx = coord(q.x), cy = coord(q.y);
  for (int ix = cx - span; ix <= cx + span; ++ix)
    for (int iy = cy - span; iy <= cy + span; ++iy) {
      auto it = cells_.find(pack(ix, iy));
      if (it == cells_.end()) continue;
      for (std::uint32_t id : it->second) {
        const V2& p = points_[id];
        if (sqnorm(p.x - q.x, p.y - q.y) <= r2) out.push_back(id);
      }
    }
  std::sort(out.begin(), out.end());
  return out;
}

// ---------------------------------------------------------------------------
// kernel.cpp:8-35
double KernelParams::sigma_tilde() const {
  return std::sqrt(sigma * sigma + sigma_eps * sigma_eps);
}
double KernelParams::moment_scale() const {
  const double st2 = sigma * sigma + sigma_eps * sigma_eps;
  return sigma * sigma / st2;
}
void KernelParams::finalize() {
  if (!(sigma > 0.0)) throw std::invalid_argument("kernel sigma must be > 0");
  if (sigma_eps < 0.0) throw std::invalid_argument("sigma_eps must be >= 0");
  if (!(lambda > 0.0)) throw std::invalid_argument("lambda must be > 0");
  cutoff_radius = std::max(cutoff_radius, 3.0 * sigma_tilde());
  if (!std::isfinite(sigma) || !std::isfinite(sigma_eps) || !std::isfinite(lambda))
    throw std::invalid_argument("non-finite kernel parameter");
}

static bool finite2(const V2& v) { return std::isfinite(v.x) && std::isfinite(v.y); }

double kernel_eval(const KernelParams& p, const V2& x, const V2& c, double bw) {
  if (!finite2(x) || !finite2(c) || !std::isfinite(bw))
    throw std::domain_error("non-finite kernel input");
  if (!(bw > 0.0)) throw std::domain_error("bandwidth must be > 0");
  const double r2 = sqnorm(x.x - c.x, x.y - c.y);
  if (r2 > p.cutoff_radius * p.cutoff_radius) return 0.0;
  return std::exp(-r2 / (2.0 * bw * bw));
}

// ---------------------------------------------------------------------------
// center_select.cpp:9-76
void TerrainObservation::validate() const {
  if (xy.size() != z.size()) throw std::invalid_argument("observation xy/z length mismatch");
  if (xy.empty()) throw std::invalid_argument("empty observation");
  for (std::size_t i = 0; i < xy.size(); ++i)
    if (!finite2(xy[i]) || !std::isfinite(z[i]))
      throw std::invalid_argument("non-finite observation coordinate");
}

std::vector<V2> supported_mesh_nodes(const TerrainObservation& pts, const Rect& roi,
                                     double res, double r_a, int count) {
  if (!(res > 0.0)) throw std::invalid_argument("mesh_resolution must be > 0");
  if (count < 1) throw std::invalid_argument("accept_count must be >= 1");
  pts.validate();
  GridIndex2 index(std::max(r_a, res));
  index.build(pts.xy);
  const int nx = static_cast<int>(std::floor((roi.max.x - roi.min.x) / res + 1e-9));
  const int ny = static_cast<int>(std::floor((roi.max.y - roi.min.y) / res + 1e-9));
  Rect bbox{pts.xy.front(), pts.xy.front()};
  for (const V2& p : pts.xy) {
    bbox.min.x = std::min(bbox.min.x, p.x);
    bbox.min.y = std::min(bbox.min.y, p.y);
    bbox.max.x = std::max(bbox.max.x, p.x);
    bbox.max.y = std::max(bbox.max.y, p.y);
  }
  bbox = bbox.dilated(r_a);
  auto clamp_idx = [&](double v, double lo, int n) {
    const int i = static_cast<int>(std::floor((v - lo) / res));
    return std::min(std::max(i, 0), n);
  };
  const int i0 = clamp_idx(bbox.min.x, roi.min.x, nx);
  const int i1 = clamp_idx(bbox.max.x, roi.min.x, nx);
  const int j0 = clamp_idx(bbox.min.y, roi.min.y, ny);
  const int j1 = clamp_idx(bbox.max.y, roi.min.y, ny);
  std::vector<V2> nodes;
  for (int i = i0; i <= i1; ++i)
    for (int j = j0; j <= j1; ++j) {
      const V2 node{roi.min.x + i * res, roi.min.y + j * res};
      if (static_cast<int>(index.radius_query(node, r_a).size()) >= count)
        nodes.push_back(node);
    }
  return nodes;
}

CenterSet select_centers(const TerrainObservation& pts, const Rect& roi, double res,
                         double r_a, int count) {
  CenterSet set;
  set.mesh_resolution = res;
  set.accept_radius = r_a;
  set.accept_count = count;
  set.roi = roi;
  set.centers = supported_mesh_nodes(pts, roi, res, r_a, count);
  if (set.centers.empty()) throw NoSupportedCenters();
  return set;
}

// ---------------------------------------------------------------------------
// Pivoted LDL^T — restates the published Eigen::LDLT algorithm (diagonal
// pivoting on the largest remaining |d|, left-looking column updates, zero
// pivots tolerated, pseudo-inverse of D in solve).
Ldlt::Ldlt(const Mat& a) : n(a.rows), lu(a), perm(static_cast<size_t>(a.rows)) {
  std::vector<double> tmp(static_cast<size_t>(n));
  bool found_zero = false;
  int sign = 0;  // 0 zero, 1 psd, 2 nsd, 3 indefinite
  for (long k = 0; k < n; ++k) {
    long big = k;
    double bv = std::abs(lu(k, k));
    for (long i = k + 1; i < n; ++i)
      if (std::abs(lu(i, i)) > bv) {
        bv = std::abs(lu(i, i));
        big = i;
      }
    perm[static_cast<size_t>(k)] = big;
    if (big != k) {
      for (long c = 0; c < k; ++c) std::swap(lu(k, c), lu(big, c));
      for (long r = big + 1; r < n; ++r) std::swap(lu(r, k), lu(r, big));
      std::swap(lu(k, k), lu(big, big));
      for (long i = k + 1; i < big; ++i) {
        const double t = lu(i, k);
        lu(i, k) = lu(big, i);
        lu(big, i) = t;
      }
    }
    if (k > 0) {
      for (long c = 0; c < k; ++c) tmp[static_cast<size_t>(c)] = lu(c, c) * lu(k, c);
      double s = 0.0;
      for (long c = 0; c < k; ++c) s += lu(k, c) * tmp[static_cast<size_t>(c)];
      lu(k, k) -= s;
      for (long r = k + 1; r < n; ++r) {
        double acc = 0.0;
        for (long c = 0; c < k; ++c) acc += lu(r, c) * tmp[static_cast<size_t>(c)];
        lu(r, k) -= acc;
      }
    }
    const double akk = lu(k, k);
    const bool valid = std::abs(akk) > 0.0;
    if (k == 0 && !valid) {
      sign = 0;
      for (long j = 0; j < n; ++j) perm[static_cast<size_t>(j)] = j;
      positive = true;
      return;
    }
    if (k + 1 < n && valid)
      for (long r = k + 1; r < n; ++r) lu(r, k) /= akk;
    else if (k + 1 < n)
      for (long r = k + 1; r < n; ++r) ok = ok && (lu(r, k) == 0.0);
    if (found_zero && valid)
      ok = false;
    else if (!valid)
      found_zero = true;
    if (sign == 1) {
      if (akk < 0.0) sign = 3;
    } else if (sign == 2) {
      if (akk > 0.0) sign = 3;
    } else if (sign == 0) {
      if (akk > 0.0) sign = 1;
      else if (akk < 0.0) sign = 2;
    }
  }
  positive = (sign == 1 || sign == 0);
}

std::vector<double> Ldlt::vectorD() const {
  std::vector<double> d(static_cast<size_t>(n));
  for (long i = 0; i < n; ++i) d[static_cast<size_t>(i)] = lu(i, i);
  return d;
}

Mat Ldlt::solve(const Mat& b) const {
  Mat x = b;
  const double tol = std::numeric_limits<double>::min();
  for (long c = 0; c < x.cols; ++c) {
    double* v = &x.a[static_cast<size_t>(c * x.rows)];
    for (long k = 0; k < n; ++k) std::swap(v[k], v[perm[static_cast<size_t>(k)]]);
    for (long k = 0; k < n; ++k)
      for (long r = k + 1; r < n; ++r) v[r] -= lu(r, k) * v[k];
    for (long k = 0; k < n; ++k) {
      const double d = lu(k, k);
      v[k] = (std::abs(d) > tol) ? v[k] / d : 0.0;
    }
    for (long k = n - 1; k >= 0; --k) {
      double s = v[k];
      for (long r = k + 1; r < n; ++r) s -= lu(r, k) * v[r];
      v[k] = s;
    }
    for (long k = n - 1; k >= 0; --k) std::swap(v[k], v[perm[static_cast<size_t>(k)]]);
  }
  return x;
}

std::vector<double> Ldlt::solve(const std::vector<double>& b) const {
  Mat m(static_cast<long>(b.size()), 1);
  m.a = b;
  return solve(m).a;
}

// ---------------------------------------------------------------------------
// terrain_model.cpp:15-22
namespace {
std::int64_t pack2(std::int64_t x, std::int64_t y) { return (x << 32) ^ (y & 0xffffffffll); }
std::int64_t mesh_node_key(const V2& node, const Rect& roi, double res) {
  return pack2(std::llround((node.x - roi.min.x) / res), std::llround((node.y - roi.min.y) / res));
}
}  // namespace

// terrain_model.cpp:26-44
TerrainModel::TerrainModel(KernelParams kernel, CenterSet centers)
    : kernel_(kernel), centers_(std::move(centers)) {
  kernel_.finalize();
  const auto n = centers_.centers.size();
  weights_.assign(n, 0.0);
  block_index_.resize(n);
  for (std::uint32_t i = 0; i < n; ++i) {
    const std::uint32_t b = block_for_tile(tile_key(centers_.centers[i]));
    block_index_[i] = b;
    blocks_[b].members.push_back(i);
  }
  for (auto& blk : blocks_) {
    const long bn = static_cast<long>(blk.members.size());
    blk.info_inv = Mat(bn, bn);
    for (long i = 0; i < bn; ++i) blk.info_inv(i, i) = 1.0 * (1.0 / kernel_.lambda);
  }
  rebuild_indexes();
}

// terrain_model.cpp:46-51
std::int64_t TerrainModel::tile_key(const V2& c) const {
  const double side = 2.0 * kernel_.cutoff_radius;
  if (!(side < 1e12)) return 0;
  return pack2(static_cast<std::int64_t>(std::floor(c.x / side)),
               static_cast<std::int64_t>(std::floor(c.y / side)));
}

// terrain_model.cpp:53-60
std::uint32_t TerrainModel::block_for_tile(std::int64_t key) {
  auto it = tile_blocks_.find(key);
  if (it != tile_blocks_.end()) return it->second;
  const auto id = static_cast<std::uint32_t>(blocks_.size());
  tile_blocks_.emplace(key, id);
  blocks_.emplace_back();
  return id;
}

// terrain_model.cpp:62-70
void TerrainModel::rebuild_indexes() {
  const double cell = std::min(kernel_.cutoff_radius, 1e6);
  center_index_ = std::make_unique<GridIndex2>(cell);
  center_index_->build(centers_.centers);
  mesh_occupancy_.clear();
  for (const V2& c : centers_.centers)
    mesh_occupancy_.emplace(mesh_node_key(c, centers_.roi, centers_.mesh_resolution), 1u);
}

std::vector<std::uint32_t> TerrainModel::centers_near(const V2& x, double radius) const {
  return center_index_->radius_query(x, radius);
}

// terrain_model.cpp:77-95
std::uint32_t TerrainModel::add_center(const V2& c) {
  const auto id = static_cast<std::uint32_t>(centers_.centers.size());
  centers_.centers.push_back(c);
  const std::uint32_t b = block_for_tile(tile_key(c));
  block_index_.push_back(b);
  Block& blk = blocks_[b];
  blk.members.push_back(id);
  const long bn = static_cast<long>(blk.members.size());
  Mat grown(bn, bn);
  for (long cc = 0; cc + 1 < bn; ++cc)
    for (long r = 0; r + 1 < bn; ++r) grown(r, cc) = blk.info_inv(r, cc);
  grown(bn - 1, bn - 1) = 1.0 / kernel_.lambda;
  blk.info_inv = std::move(grown);
  weights_.push_back(0.0);
  center_index_->insert(c);
  mesh_occupancy_.emplace(mesh_node_key(c, centers_.roi, centers_.mesh_resolution), 1u);
  return id;
}

// terrain_model.cpp:97-107
SparseVec TerrainModel::moment_feature(const V2& x) const {
  if (!finite2(x)) throw std::domain_error("non-finite query");
  SparseVec m;
  const double scale = kernel_.moment_scale();
  const double st = kernel_.sigma_tilde();
  for (std::uint32_t id : centers_near(x, kernel_.cutoff_radius)) {
    const double k = kernel_eval(kernel_, x, centers_.centers[id], st);
    if (k != 0.0) m.entries.emplace_back(id, scale * k);
  }
  return m;
}

// terrain_model.cpp:109-125 (single 256-chunk of parallel.hpp:31-45: acc = 0 + s)
HeightQuery TerrainModel::predict_height(const V2& x) const {
  const auto ids = centers_near(x, kernel_.cutoff_radius);
  if (ids.empty()) return {0.0, false};
  double acc = 0.0;
  for (std::size_t b = 0; b < ids.size(); b += 256) {
    const std::size_t e = std::min(ids.size(), b + 256);
    double s = 0.0;
    for (std::size_t i = b; i < e; ++i)
      s += weights_[ids[i]] * kernel_eval(kernel_, x, centers_.centers[ids[i]], kernel_.sigma);
    acc += s;
  }
  return {acc, true};
}

// terrain_model.cpp:127-143; element order (w * ((-(x-c)) * inv_s2)) * k
V2 TerrainModel::predict_gradient(const V2& x) const {
  const auto ids = centers_near(x, kernel_.cutoff_radius);
  const double inv_s2 = 1.0 / (kernel_.sigma * kernel_.sigma);
  V2 acc{0.0, 0.0};
  for (std::size_t b = 0; b < ids.size(); b += 256) {
    const std::size_t e = std::min(ids.size(), b + 256);
    V2 s{0.0, 0.0};
    for (std::size_t i = b; i < e; ++i) {
      const V2& c = centers_.centers[ids[i]];
      const double k = kernel_eval(kernel_, x, c, kernel_.sigma);
      const double w = weights_[ids[i]];
      s.x += (w * ((-(x.x - c.x)) * inv_s2)) * k;
      s.y += (w * ((-(x.y - c.y)) * inv_s2)) * k;
    }
    acc.x += s.x;
    acc.y += s.y;
  }
  return acc;
}

// terrain_model.cpp:145-253
UpdateReport TerrainModel::recursive_update(const TerrainObservation& obs, bool allow_birth) {
  obs.validate();
  UpdateReport report;
  if (allow_birth) {
    const auto nodes = supported_mesh_nodes(obs, centers_.roi, centers_.mesh_resolution,
                                            centers_.accept_radius, centers_.accept_count);
    for (const V2& node : nodes) {
      const auto key = mesh_node_key(node, centers_.roi, centers_.mesh_resolution);
      if (mesh_occupancy_.count(key)) continue;
      add_center(node);
      ++report.born_centers;
    }
  }
  std::vector<char> active(centers_.centers.size(), 0);
  for (const V2& x : obs.xy)
    for (std::uint32_t id : centers_near(x, kernel_.cutoff_radius)) active[id] = 1;
  std::set<std::uint32_t> active_blocks;
  for (std::uint32_t i = 0; i < active.size(); ++i)
    if (active[i]) active_blocks.insert(block_index_[i]);
  report.active_blocks = active_blocks.size();
  if (active_blocks.empty()) return report;

  std::vector<std::uint32_t> merged;
  for (std::uint32_t b : active_blocks)
    merged.insert(merged.end(), blocks_[b].members.begin(), blocks_[b].members.end());
  report.active_centers = merged.size();
  const long n = static_cast<long>(merged.size());
  const long m_total = static_cast<long>(obs.size());
  std::vector<std::int32_t> row_of(centers_.centers.size(), -1);
  for (long r = 0; r < n; ++r) row_of[merged[static_cast<size_t>(r)]] = static_cast<std::int32_t>(r);

  Mat Mt(n, m_total);
  const double scale = kernel_.moment_scale();
  const double st = kernel_.sigma_tilde();
  for (long j = 0; j < m_total; ++j) {
    const V2& x = obs.xy[static_cast<size_t>(j)];
    for (std::uint32_t id : centers_near(x, kernel_.cutoff_radius)) {
      const double k = kernel_eval(kernel_, x, centers_.centers[id], st);
      if (k != 0.0) Mt(row_of[id], j) = scale * k;
    }
  }
  Mat Hinv(n, n);
  std::vector<double> w(static_cast<size_t>(n));
  {
    long off = 0;
    for (std::uint32_t b : active_blocks) {
      const long bn = static_cast<long>(blocks_[b].members.size());
      for (long c = 0; c < bn; ++c)
        for (long r = 0; r < bn; ++r) Hinv(off + r, off + c) = blocks_[b].info_inv(r, c);
      for (long i = 0; i < bn; ++i)
        w[static_cast<size_t>(off + i)] = weights_[blocks_[b].members[static_cast<size_t>(i)]];
      off += bn;
    }
  }
  constexpr long kChunk = 64;
  for (long o = 0; o < m_total; o += kChunk) {
    const long m = std::min(kChunk, m_total - o);
    // K = Hinv * Mc  (n x m)
    Mat K(n, m);
    for (long c = 0; c < m; ++c)
      for (long k = 0; k < n; ++k) {
        const double v = Mt(k, o + c);
        if (v == 0.0) continue;
        for (long r = 0; r < n; ++r) K(r, c) += Hinv(r, k) * v;
      }
    // S = Mc^T K + I, symmetrised
    Mat S(m, m);
    for (long c = 0; c < m; ++c)
      for (long r = 0; r < m; ++r) {
        double s = 0.0;
        for (long k = 0; k < n; ++k) s += Mt(k, o + r) * K(k, c);
        S(r, c) = s;
      }
    for (long i = 0; i < m; ++i) S(i, i) += 1.0;
    Mat Ss(m, m);
    for (long c = 0; c < m; ++c)
      for (long r = 0; r < m; ++r) Ss(r, c) = 0.5 * (S(r, c) + S(c, r));
    Ldlt ldlt(Ss);
    if (!ldlt.ok || !ldlt.positive) {
      report.rejected = true;
      return report;
    }
    Mat Kt(m, n);
    for (long c = 0; c < n; ++c)
      for (long r = 0; r < m; ++r) Kt(r, c) = K(c, r);
    const Mat KS = ldlt.solve(Kt);  // m x n
    for (double v : KS.a)
      if (!std::isfinite(v)) {
        report.rejected = true;
        return report;
      }
    // Hinv -= K * KS
    for (long c = 0; c < n; ++c)
      for (long k = 0; k < m; ++k) {
        const double v = KS(k, c);
        for (long r = 0; r < n; ++r) Hinv(r, c) -= K(r, k) * v;
      }
    for (long c = 0; c < n; ++c)
      for (long r = c + 1; r < n; ++r) {
        const double s = 0.5 * (Hinv(r, c) + Hinv(c, r));
        Hinv(r, c) = s;
        Hinv(c, r) = s;
      }
    // resid = z_c - Mc^T w ; w += Hinv * (Mc * resid)
    std::vector<double> resid(static_cast<size_t>(m));
    for (long r = 0; r < m; ++r) {
      double s = 0.0;
      for (long k = 0; k < n; ++k) s += Mt(k, o + r) * w[static_cast<size_t>(k)];
      resid[static_cast<size_t>(r)] = obs.z[static_cast<size_t>(o + r)] - s;
    }
    std::vector<double> mr(static_cast<size_t>(n), 0.0);
    for (long c = 0; c < m; ++c)
      for (long k = 0; k < n; ++k) mr[static_cast<size_t>(k)] += Mt(k, o + c) * resid[static_cast<size_t>(c)];
    std::vector<double> dw(static_cast<size_t>(n), 0.0);
    for (long c = 0; c < n; ++c) {
      const double v = mr[static_cast<size_t>(c)];
      for (long r = 0; r < n; ++r) dw[static_cast<size_t>(r)] += Hinv(r, c) * v;
    }
    for (long r = 0; r < n; ++r) w[static_cast<size_t>(r)] += dw[static_cast<size_t>(r)];
  }
  {
    long off = 0;
    for (std::uint32_t b : active_blocks) {
      const long bn = static_cast<long>(blocks_[b].members.size());
      Mat blk(bn, bn);
      for (long c = 0; c < bn; ++c)
        for (long r = 0; r < bn; ++r) blk(r, c) = Hinv(off + r, off + c);
      Mat sym(bn, bn);
      for (long c = 0; c < bn; ++c)
        for (long r = 0; r < bn; ++r) sym(r, c) = 0.5 * (blk(r, c) + blk(c, r));
      blocks_[b].info_inv = std::move(sym);
      for (long i = 0; i < bn; ++i)
        weights_[blocks_[b].members[static_cast<size_t>(i)]] = w[static_cast<size_t>(off + i)];
      off += bn;
    }
  }
  return report;
}

// terrain_model.cpp:269-308
TerrainModel fit_batch_ridge(const KernelParams& params, const CenterSet& centers,
                             const TerrainObservation& obs) {
  obs.validate();
  TerrainModel model(params, centers);
  const long n = static_cast<long>(model.num_centers());
  Mat H(n, n);
  for (long i = 0; i < n; ++i) H(i, i) = 1.0 * model.kernel().lambda;
  std::vector<double> b(static_cast<size_t>(n), 0.0);
  for (std::size_t j = 0; j < obs.size(); ++j) {
    const SparseVec m = model.moment_feature(obs.xy[j]);
    for (const auto& [i1, v1] : m.entries) {
      b[i1] += v1 * obs.z[j];
      for (const auto& [i2, v2] : m.entries) H(i1, i2) += v1 * v2;
    }
  }
  Ldlt ldlt(H);
  std::vector<double> w = ldlt.solve(b);
  bool finite = true;
  for (double v : w) finite = finite && std::isfinite(v);
  if (!ldlt.ok || !finite) {
    const auto d = ldlt.vectorD();
    double mx = 0.0, mn = std::numeric_limits<double>::infinity();
    for (double v : d) {
      mx = std::max(mx, std::abs(v));
      mn = std::min(mn, std::abs(v));
    }
    throw std::runtime_error("ridge solve failed; condition estimate " +
                             std::to_string(mx / std::max(mn, 1e-300)));
  }
  model.weights_ = w;
  for (auto& blk : model.blocks_) {
    const long bn = static_cast<long>(blk.members.size());
    Mat Hb(bn, bn), I(bn, bn);
    for (long r = 0; r < bn; ++r) {
      I(r, r) = 1.0;
      for (long c = 0; c < bn; ++c) Hb(r, c) = H(blk.members[static_cast<size_t>(r)], blk.members[static_cast<size_t>(c)]);
    }
    const Mat inv = Ldlt(Hb).solve(I);
    Mat sym(bn, bn);
    for (long c = 0; c < bn; ++c)
      for (long r = 0; r < bn; ++r) sym(r, c) = 0.5 * (inv(r, c) + inv(c, r));
    blk.info_inv = std::move(sym);
  }
  return model;
}

// ---------------------------------------------------------------------------
// snapshot.cpp:7-126 ("RBFT" v1, little-endian)
namespace {
template <typename T>
void put(std::ostream& out, const T& v) {
  out.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <typename T>
T get(std::istream& in) {
  T v;
  in.read(reinterpret_cast<char*>(&v), sizeof(T));
  if (!in) throw std::runtime_error("truncated terrain snapshot");
  return v;
}
}  // namespace

void TerrainModel::save(const std::string& path) const {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot open " + path);
  out.write("RBFT", 4);
  put<std::uint32_t>(out, 1u);
  put<std::uint32_t>(out, static_cast<std::uint32_t>(num_centers()));
  put<std::uint32_t>(out, static_cast<std::uint32_t>(blocks_.size()));
  for (const V2& c : centers_.centers) {
    put<double>(out, c.x);
    put<double>(out, c.y);
  }
  for (double w : weights_) put<double>(out, w);
  for (std::uint32_t b : block_index_) put<std::uint32_t>(out, b);
  for (const Block& blk : blocks_)
    for (long r = 0; r < blk.info_inv.rows; ++r)
      for (long c = 0; c <= r; ++c) put<double>(out, blk.info_inv(r, c));
  put<double>(out, kernel_.sigma);
  put<double>(out, kernel_.sigma_eps);
  put<double>(out, kernel_.lambda);
  put<double>(out, kernel_.cutoff_radius);
  put<double>(out, centers_.mesh_resolution);
  put<double>(out, centers_.accept_radius);
  put<std::uint32_t>(out, static_cast<std::uint32_t>(centers_.accept_count));
  put<double>(out, centers_.roi.min.x);
  put<double>(out, centers_.roi.min.y);
  put<double>(out, centers_.roi.max.x);
  put<double>(out, centers_.roi.max.y);
}

TerrainModel TerrainModel::load(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open " + path);
  char magic[4];
  in.read(magic, 4);
  if (!in || std::memcmp(magic, "RBFT", 4) != 0)
    throw std::runtime_error("not a terrain snapshot: " + path);
  if (get<std::uint32_t>(in) != 1u) throw std::runtime_error("unsupported snapshot version");
  const auto n = get<std::uint32_t>(in);
  const auto nb = get<std::uint32_t>(in);
  TerrainModel model;
  model.centers_.centers.resize(n);
  for (auto& c : model.centers_.centers) {
    c.x = get<double>(in);
    c.y = get<double>(in);
  }
  model.weights_.resize(n);
  for (std::uint32_t i = 0; i < n; ++i) model.weights_[i] = get<double>(in);
  model.block_index_.resize(n);
  model.blocks_.resize(nb);
  for (std::uint32_t i = 0; i < n; ++i) {
    const auto b = get<std::uint32_t>(in);
    if (b >= nb) throw std::runtime_error("corrupt block index");
    model.block_index_[i] = b;
    model.blocks_[b].members.push_back(i);
  }
  for (auto& blk : model.blocks_) {
    const long bn = static_cast<long>(blk.members.size());
    blk.info_inv = Mat(bn, bn);
    for (long r = 0; r < bn; ++r)
      for (long c = 0; c <= r; ++c) {
        const double v = get<double>(in);
        blk.info_inv(r, c) = v;
        blk.info_inv(c, r) = v;
      }
  }
  model.kernel_.sigma = get<double>(in);
  model.kernel_.sigma_eps = get<double>(in);
  model.kernel_.lambda = get<double>(in);
  model.kernel_.cutoff_radius = get<double>(in);
  model.centers_.mesh_resolution = get<double>(in);
  model.centers_.accept_radius = get<double>(in);
  model.centers_.accept_count = static_cast<int>(get<std::uint32_t>(in));
  model.centers_.roi.min.x = get<double>(in);
  model.centers_.roi.min.y = get<double>(in);
  model.centers_.roi.max.x = get<double>(in);
  model.centers_.roi.max.y = get<double>(in);
  model.kernel_.finalize();
  for (std::uint32_t i = 0; i < n; ++i)
    model.tile_blocks_.emplace(model.tile_key(model.centers_.centers[i]), model.block_index_[i]);
  model.rebuild_indexes();
  return model;
}

// ---------------------------------------------------------------------------
// so3.cpp:8-27
M3 hat(const V3& v) {
  M3 m;
  m.a[0] = 0.0;  m.a[1] = -v.z; m.a[2] = v.y;
  m.a[3] = v.z;  m.a[4] = 0.0;  m.a[5] = -v.x;
  m.a[6] = -v.y; m.a[7] = v.x;  m.a[8] = 0.0;
  return m;
}

M3 mul(const M3& a, const M3& b) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = (a(i, 0) * b(0, j) + a(i, 1) * b(1, j)) + a(i, 2) * b(2, j);
  return r;
}

V3 mul(const M3& a, const V3& v) {
  return {(a(0, 0) * v.x + a(0, 1) * v.y) + a(0, 2) * v.z,
          (a(1, 0) * v.x + a(1, 1) * v.y) + a(1, 2) * v.z,
          (a(2, 0) * v.x + a(2, 1) * v.y) + a(2, 2) * v.z};
}

M3 so3_exp(const V3& w) {
  const double theta2 = (w.x * w.x + w.y * w.y) + w.z * w.z;
  const M3 W = hat(w);
  const M3 W2 = mul(W, W);
  M3 R;
  if (theta2 < 1e-16) {
    for (int i = 0; i < 9; ++i) R.a[i] = ((i % 4 == 0) ? 1.0 : 0.0) + W.a[i] + 0.5 * W2.a[i];
    return R;
  }
  const double theta = std::sqrt(theta2);
  const double a = std::sin(theta) / theta;
  const double b = (1.0 - std::cos(theta)) / theta2;
  for (int i = 0; i < 9; ++i) R.a[i] = ((i % 4 == 0) ? 1.0 : 0.0) + a * W.a[i] + b * W2.a[i];
  return R;
}

// ---------------------------------------------------------------------------
// contact.cpp:7-39 (residual + 1x6 Jacobian) with the scan_matcher.cpp:
// 221-248 weighting: sqrt(lambda_M) * w_Huber, invalid rows stay zero.
ManifoldRow manifold_row(const TerrainModel& terrain, const M3& R, const V3& t, const V3& h,
                         double wheel_radius, double lambda_M, double huber_delta) {
  ManifoldRow row;
  const V3 Rh = mul(R, h);
  const V3 xi{Rh.x + t.x, Rh.y + t.y, Rh.z + t.z};
  const HeightQuery q = terrain.predict_height({xi.x, xi.y});
  if (!q.supported) return row;
  row.valid = true;
  row.raw = xi.z - wheel_radius - q.z;
  const V2 grad = terrain.predict_gradient({xi.x, xi.y});
  const double dr[3] = {-grad.x, -grad.y, 1.0};
  // dxi/dtheta = (-R) * hat(h)
  M3 negR;
  for (int i = 0; i < 9; ++i) negR.a[i] = -R.a[i];
  const M3 D = mul(negR, hat(h));
  double J[6];
  for (int c = 0; c < 3; ++c) J[c] = (dr[0] * D(0, c) + dr[1] * D(1, c)) + dr[2] * D(2, c);
  J[3] = dr[0];
  J[4] = dr[1];
  J[5] = dr[2];
  const double sl = std::sqrt(lambda_M);
  double w = 1.0;
  if (huber_delta > 0.0 && std::abs(row.raw) > huber_delta)
    w = std::sqrt(huber_delta / std::abs(row.raw));
  row.r = sl * w * row.raw;
  for (int c = 0; c < 6; ++c) row.J[c] = sl * w * J[c];
  return row;
}

void accumulate(NormalEq& ne, const ManifoldRow& row) {
  for (int i = 0; i < 6; ++i) {
    for (int j = 0; j < 6; ++j) ne.A[6 * i + j] += row.J[i] * row.J[j];
    ne.g[i] += row.J[i] * row.r;
  }
  ne.cost += row.r * row.r;
  ne.valid += row.valid ? 1 : 0;
}

bool lm_step(const NormalEq& ne, double mu, double delta[6]) {
  Mat damped(6, 6);
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) damped(i, j) = ne.A[6 * i + j];
  for (int i = 0; i < 6; ++i) damped(i, i) += mu * std::max(ne.A[6 * i + i], 1e-12);
  for (int i = 0; i < 6; ++i) damped(i, i) += 1e-3;
  std::vector<double> g(ne.g, ne.g + 6);
  const auto x = Ldlt(damped).solve(g);
  bool finite = true;
  for (int i = 0; i < 6; ++i) {
    delta[i] = -x[static_cast<size_t>(i)];
    finite = finite && std::isfinite(delta[i]);
  }
  return finite;
}

// --- pipeline.cpp:150-170 ----------------------------------------------------
GroundPoints select_ground_points(const std::vector<V3>& p, const std::vector<std::uint8_t>& kind,
                                  const M3& R, const V3& t, const Rect& roi, double radius,
                                  double voxel, std::size_t max_points) {
  GroundPoints out;
  std::unordered_set<std::int64_t> voxels;
  for (std::size_t i = 0; i < p.size(); ++i) {
    if (kind[i] != 2) continue;  // FeatureKind::Ground
    const V3 q0 = mul(R, p[i]);
    const V3 q{q0.x + t.x, q0.y + t.y, q0.z + t.z};
    const V2 xy{q.x, q.y};
    if (!roi.contains(xy)) continue;
    if (std::sqrt(sqnorm(xy.x - t.x, xy.y - t.y)) > radius) continue;
    const auto vx = static_cast<std::int64_t>(std::floor(xy.x / voxel));
    const auto vy = static_cast<std::int64_t>(std::floor(xy.y / voxel));
    if (!voxels.insert((vx << 21) ^ (vy & ((1 << 21) - 1))).second) continue;
    out.xy.push_back(xy);
    out.z.push_back(q.z);
    if (out.xy.size() >= max_points) break;
  }
  return out;
}

// --- metrics.cpp:199-232 -------------------------------------------------------
Histogram terrain_error_histogram(const TerrainModel& model, const std::vector<V2>& xy,
                                  const std::vector<double>& z, double trim_fraction, int bins) {
  if (xy.empty() || xy.size() != z.size())
    throw std::invalid_argument("histogram needs matched non-empty samples");
  if (trim_fraction < 0.0 || trim_fraction >= 1.0)
    throw std::invalid_argument("trim_fraction must be in [0, 1)");
  constexpr double kRange = 0.25;
  std::vector<double> errors(xy.size());
  for (std::size_t i = 0; i < xy.size(); ++i) {
    const HeightQuery q = model.predict_height(xy[i]);
    errors[i] = q.supported ? std::abs(z[i] - q.z) : kRange;
  }
  std::sort(errors.begin(), errors.end());
  const std::size_t keep =
      xy.size() - static_cast<std::size_t>(std::floor(trim_fraction * static_cast<double>(xy.size())));
  Histogram h;
  h.trimmed = xy.size() - keep;
  h.edges.resize(bins + 1);
  h.counts.assign(bins, 0);
  for (int b = 0; b <= bins; ++b) h.edges[b] = kRange * b / bins;
  for (std::size_t i = 0; i < keep; ++i) {
    const auto b = static_cast<int>(std::floor(errors[i] / kRange * bins));
    if (b >= bins)
      ++h.overflow;
    else
      ++h.counts[b];
  }
  return h;
}

// --- terrain_model.cpp:255-267 -------------------------------------------------
void export_grid(const TerrainModel& model, double grid_step, std::vector<double>& xs,
                 std::vector<double>& ys, std::vector<double>& zs) {
  const Rect& roi = model.centers().roi;
  for (double x = roi.min.x; x <= roi.max.x + 1e-12; x += grid_step) {
    for (double y = roi.min.y; y <= roi.max.y + 1e-12; y += grid_step) {
      const HeightQuery q = model.predict_height({x, y});
      if (!q.supported) continue;
      xs.push_back(x);
      ys.push_back(y);
      zs.push_back(q.z);
    }
  }
}

// --- local_map.cpp:8-62 --------------------------------------------------------
static std::int64_t map_voxel_key(const V3& p, double size) {
  auto q = [&](double v) { return static_cast<std::int64_t>(std::floor(v / size)) & 0x1fffff; };
  return (q(p.x) << 42) | (q(p.y) << 21) | q(p.z);
}

void LocalMap::insert(const FeatureInput& scan, const M3& R, const V3& t) {
  Frame fr;
  std::unordered_set<std::int64_t> edge_seen, planar_seen;
  for (std::size_t i = 0; i < scan.p.size(); ++i) {
    const V3 q0 = mul(R, scan.p[i]);
    const V3 p{q0.x + t.x, q0.y + t.y, q0.z + t.z};
    if (scan.kind[i] == 0) {
      if (cfg_.voxel_size > 0.0 && !edge_seen.insert(map_voxel_key(p, cfg_.voxel_size)).second)
        continue;
      fr.edge.push_back(p);
      fr.edge_label.push_back(scan.label[i]);
    } else {
      if (cfg_.voxel_size > 0.0 && !planar_seen.insert(map_voxel_key(p, cfg_.voxel_size)).second)
        continue;
      fr.planar.push_back(p);
      fr.planar_label.push_back(scan.label[i]);
    }
  }
  frames_.push_back(std::move(fr));
  while (frames_.size() > cfg_.window) frames_.erase(frames_.begin());
  edge.clear();
  planar.clear();
  edge_label.clear();
  planar_label.clear();
  for (const Frame& f : frames_) {
    edge.insert(edge.end(), f.edge.begin(), f.edge.end());
    planar.insert(planar.end(), f.planar.begin(), f.planar.end());
    edge_label.insert(edge_label.end(), f.edge_label.begin(), f.edge_label.end());
    planar_label.insert(planar_label.end(), f.planar_label.begin(), f.planar_label.end());
  }
  edge_tree.build(edge);
  planar_tree.build(planar);
}

// kdtree.hpp:31-41/:79-99: the k smallest (d2, id) with d2 <= gate^2, ascending
std::vector<std::uint32_t> knn(const std::vector<V3>& pts, const V3& q, int k, double gate) {
  const double gate2 = gate * gate;
  std::vector<std::pair<double, std::uint32_t>> cand;
  for (std::uint32_t i = 0; i < pts.size(); ++i) {
    const double dx = pts[i].x - q.x, dy = pts[i].y - q.y, dz = pts[i].z - q.z;
    const double d2 = (dx * dx + dy * dy) + dz * dz;
    if (d2 <= gate2) cand.emplace_back(d2, i);
  }
  const std::size_t m = std::min<std::size_t>(cand.size(), static_cast<std::size_t>(k));
  std::partial_sort(cand.begin(), cand.begin() + m, cand.end());
  std::vector<std::uint32_t> out(m);
  for (std::size_t i = 0; i < m; ++i) out[i] = cand[i].second;
  return out;
}

static double coord(const V3& p, int axis) { return axis == 0 ? p.x : (axis == 1 ? p.y : p.z); }

void KdTree3::build(const std::vector<V3>& pts) {
  pts_ = pts;
  order_.resize(pts.size());
  for (std::uint32_t i = 0; i < pts.size(); ++i) order_[i] = i;
  nodes_.clear();
  nodes_.reserve(pts.size());
  root_ = pts.empty() ? -1 : build_range(0, static_cast<int>(pts.size()), 0);
}

int KdTree3::build_range(int b, int e, int depth) {
  if (b >= e) return -1;
  const int axis = depth % 3, mid = (b + e) / 2;
  std::nth_element(order_.begin() + b, order_.begin() + mid, order_.begin() + e,
                   [&](std::uint32_t a, std::uint32_t c) {
                     const double va = coord(pts_[a], axis), vc = coord(pts_[c], axis);
                     return va != vc ? va < vc : a < c;
                   });
  const int self = static_cast<int>(nodes_.size());
  nodes_.push_back({order_[mid], -1, -1, axis});
  const int l = build_range(b, mid, depth + 1);
  const int r = build_range(mid + 1, e, depth + 1);
  nodes_[self].left = l;
  nodes_[self].right = r;
  return self;
}

void KdTree3::search(int ni, const V3& q, int k, double gate2,
                     std::vector<std::pair<double, std::uint32_t>>& heap) const {
  const Node& n = nodes_[ni];
  const V3& p = pts_[n.id];
  const double dx = p.x - q.x, dy = p.y - q.y, dz = p.z - q.z;
  const double d2 = (dx * dx + dy * dy) + dz * dz;
  if (d2 <= gate2) {
    const std::pair<double, std::uint32_t> c{d2, n.id};
    if (static_cast<int>(heap.size()) < k) {
      heap.push_back(c);
      std::push_heap(heap.begin(), heap.end());
    } else if (c < heap.front()) {
      std::pop_heap(heap.begin(), heap.end());
      heap.back() = c;
      std::push_heap(heap.begin(), heap.end());
    }
  }
  const double delta = coord(q, n.axis) - coord(p, n.axis);
  const int near = delta < 0 ? n.left : n.right, far = delta < 0 ? n.right : n.left;
  if (near >= 0) search(near, q, k, gate2, heap);
  const double worst =
      static_cast<int>(heap.size()) < k ? gate2 : std::min(gate2, heap.front().first);
  if (far >= 0 && delta * delta <= worst) search(far, q, k, gate2, heap);
}

std::vector<std::uint32_t> KdTree3::knn(const V3& q, int k, double gate) const {
  std::vector<std::pair<double, std::uint32_t>> heap;
  if (root_ >= 0) search(root_, q, k, gate * gate, heap);
  std::sort_heap(heap.begin(), heap.end());
  std::vector<std::uint32_t> out(heap.size());
  for (std::size_t i = 0; i < heap.size(); ++i) out[i] = heap[i].second;
  return out;
}

// cyclic Jacobi on a symmetric 3x3 (row-major in, column-major vectors out)
void eigen_sym3(const double A[9], double evals[3], double evecs[9]) {
  double a[3][3], v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) a[i][j] = A[3 * i + j];
  for (int sweep = 0; sweep < 60; ++sweep) {
    const double off = std::fabs(a[0][1]) + std::fabs(a[0][2]) + std::fabs(a[1][2]);
    if (off == 0.0) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (a[p][q] == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        const double tt = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(tt * tt + 1.0), sn = tt * c;
        for (int r = 0; r < 3; ++r) {  // A <- A G
          const double arp = a[r][p], arq = a[r][q];
          a[r][p] = c * arp - sn * arq;
          a[r][q] = sn * arp + c * arq;
        }
        for (int r = 0; r < 3; ++r) {  // A <- G^T A
          const double apr = a[p][r], aqr = a[q][r];
          a[p][r] = c * apr - sn * aqr;
          a[q][r] = sn * apr + c * aqr;
        }
        a[p][q] = a[q][p] = 0.0;
        for (int r = 0; r < 3; ++r) {
          const double vrp = v[r][p], vrq = v[r][q];
          v[r][p] = c * vrp - sn * vrq;
          v[r][q] = sn * vrp + c * vrq;
        }
      }
  }
  int idx[3] = {0, 1, 2};  // stable insertion sort, ascending eigenvalues
  for (int i = 1; i < 3; ++i)
    for (int j = i; j > 0 && a[idx[j]][idx[j]] < a[idx[j - 1]][idx[j - 1]]; --j)
      std::swap(idx[j], idx[j - 1]);
  for (int c = 0; c < 3; ++c) {
    evals[c] = a[idx[c]][idx[c]];
    for (int r = 0; r < 3; ++r) evecs[3 * c + r] = v[r][idx[c]];
  }
}

// scan_matcher.cpp:21-33
static std::int32_t majority_label(const std::vector<std::int32_t>& labels) {
  std::map<std::int32_t, int> counts;
  for (auto l : labels) ++counts[l];
  std::int32_t best = -1;
  int best_n = 0;
  for (const auto& [l, n] : counts)
    if (n > best_n) {
      best = l;
      best_n = n;
    }
  return best;
}

static V3 normalized(const V3& v) {
  const double n = std::sqrt((v.x * v.x + v.y * v.y) + v.z * v.z);
  return {v.x / n, v.y / n, v.z / n};
}

// residuals.cpp:7-25
static V3 line_residual(const V3& p, const V3& q, const V3& d, double J[9]) {
  const double dd[3] = {d.x, d.y, d.z};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) J[3 * i + j] = (i == j ? 1.0 : 0.0) - dd[i] * dd[j];
  const double e[3] = {p.x - q.x, p.y - q.y, p.z - q.z};
  V3 r;
  double* rr[3] = {&r.x, &r.y, &r.z};
  for (int i = 0; i < 3; ++i) *rr[i] = (J[3 * i] * e[0] + J[3 * i + 1] * e[1]) + J[3 * i + 2] * e[2];
  return r;
}
static double plane_residual(const V3& p, const V3& n, double offset) {
  return ((n.x * p.x + n.y * p.y) + n.z * p.z) + offset;
}
static double norm3(const V3& v) { return std::sqrt((v.x * v.x + v.y * v.y) + v.z * v.z); }

// scan_matcher.cpp:44-183
std::vector<Correspondence> build_correspondences(const FeatureInput& f, const M3& R, const V3& t,
                                                  const LocalMap& map, const SolverConfigM& cfg) {
  std::vector<Correspondence> out;
  if (map.edge.empty() && map.planar.empty()) return out;
  std::set<std::pair<std::int64_t, std::int64_t>> ground_cells;
  for (std::uint32_t i = 0; i < f.p.size(); ++i) {
    const V3 q0 = mul(R, f.p[i]);
    const V3 pw{q0.x + t.x, q0.y + t.y, q0.z + t.z};
    if (f.kind[i] == 2) {
      if (cfg.ground_corr_radius > 0.0 &&
          std::sqrt(sqnorm(pw.x - t.x, pw.y - t.y)) > cfg.ground_corr_radius)
        continue;
      if (cfg.ground_corr_voxel > 0.0) {
        const double v = cfg.ground_corr_voxel;
        const auto cell = std::make_pair(static_cast<std::int64_t>(std::floor(pw.x / v)),
                                         static_cast<std::int64_t>(std::floor(pw.y / v)));
        if (!ground_cells.insert(cell).second) continue;
      }
    }
    const bool edge = f.kind[i] == 0;
    const std::vector<V3>& pts = edge ? map.edge : map.planar;
    const std::vector<std::int32_t>& lab = edge ? map.edge_label : map.planar_label;
    const int k = edge ? 5 : 8;
    if (pts.empty()) continue;
    const auto nn = map.use_tree ? (edge ? map.edge_tree : map.planar_tree).knn(pw, k, cfg.corr_gate)
                                 : knn(pts, pw, k, cfg.corr_gate);
    if (static_cast<int>(nn.size()) < k) continue;
    V3 cen{0.0, 0.0, 0.0};
    for (auto id : nn) {
      cen.x += pts[id].x;
      cen.y += pts[id].y;
      cen.z += pts[id].z;
    }
    cen = {cen.x / nn.size(), cen.y / nn.size(), cen.z / nn.size()};
    double S[9] = {0};
    std::vector<std::int32_t> labels;
    for (auto id : nn) {
      const double d[3] = {pts[id].x - cen.x, pts[id].y - cen.y, pts[id].z - cen.z};
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) S[3 * a + b] += d[a] * d[b];
      labels.push_back(lab[id]);
    }
    double ev[3], evec[9];
    eigen_sym3(S, ev, evec);
    Correspondence c;
    c.feature = i;
    c.p_sensor = f.p[i];
    c.label = majority_label(labels);
    if (edge) {
      if (ev[2] < cfg.edge_eig_ratio * std::max(ev[1], 1e-12)) continue;
      if (ev[2] < cfg.edge_min_extent * cfg.edge_min_extent) continue;
      c.kind = 0;
      c.line_point = cen;
      c.line_dir = normalized({evec[6], evec[7], evec[8]});
      bool on_line = true;
      double J[9];
      for (auto id : nn)
        if (norm3(line_residual(pts[id], c.line_point, c.line_dir, J)) > cfg.edge_fit_tol) {
          on_line = false;
          break;
        }
      if (!on_line) continue;
      const double dist = norm3(line_residual(pw, c.line_point, c.line_dir, J));
      if (dist > cfg.corr_gate) continue;
      if (cfg.huber_delta > 0.0 && dist > cfg.huber_delta) c.weight = cfg.huber_delta / dist;
      c.dist = dist;
      c.fitq = 0.0;
    } else {
      if (ev[1] < cfg.plane_eig_ratio * ev[0] || ev[1] < 1e-3) continue;
      if (ev[2] > 50.0 * ev[1]) continue;
      c.kind = 1;
      c.normal = normalized({evec[0], evec[1], evec[2]});
      c.offset = -((c.normal.x * cen.x + c.normal.y * cen.y) + c.normal.z * cen.z);
      bool flat = true;
      for (auto id : nn)
        if (std::fabs(plane_residual(pts[id], c.normal, c.offset)) > cfg.plane_fit_tol) {
          flat = false;
          break;
        }
      if (!flat) continue;
      const double dist = std::fabs(plane_residual(pw, c.normal, c.offset));
      if (dist > cfg.corr_gate) continue;
      if (cfg.huber_delta > 0.0 && dist > cfg.huber_delta) c.weight = cfg.huber_delta / dist;
      c.dist = dist;
      c.fitq = ev[0];
    }
    out.push_back(c);
  }
  if (cfg.trim_ratio > 0.0 && !out.empty()) {
    std::vector<double> d;
    for (const auto& c : out) d.push_back(c.dist);
    std::nth_element(d.begin(), d.begin() + d.size() / 2, d.end());
    const double cut = std::max(cfg.trim_ratio * d[d.size() / 2], cfg.trim_floor);
    double qcut = std::numeric_limits<double>::infinity();
    std::vector<double> pq;
    for (const auto& c : out)
      if (c.kind == 1) pq.push_back(c.fitq);
    if (!pq.empty()) {
      std::nth_element(pq.begin(), pq.begin() + pq.size() / 2, pq.end());
      qcut = std::max(10.0 * pq[pq.size() / 2], 1e-7);
    }
    std::vector<Correspondence> kept;
    for (const auto& c : out)
      if (c.dist <= cut && c.fitq <= qcut) kept.push_back(c);
    out = std::move(kept);
  }
  return out;
}

// scan_matcher.cpp:185-216 feature rows: p = R p_s + t, dp = [-R hat(p_s), I]
void feature_normal_eq(const std::vector<Correspondence>& cs, const M3& R, const V3& t,
                       NormalEq& ne, std::size_t* rows) {
  std::size_t nr = 0;
  for (const auto& c : cs) {
    const V3 q0 = mul(R, c.p_sensor);
    const V3 pw{q0.x + t.x, q0.y + t.y, q0.z + t.z};
    const M3 H = hat(c.p_sensor);
    double dp[3][6];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        dp[i][j] = (-R(i, 0) * H(0, j) + -R(i, 1) * H(1, j)) + -R(i, 2) * H(2, j);
        dp[i][3 + j] = (i == j) ? 1.0 : 0.0;
      }
    const double sw = std::sqrt(c.weight);
    if (c.kind == 0) {
      double J[9];
      const V3 r = line_residual(pw, c.line_point, c.line_dir, J);
      const double rv[3] = {r.x, r.y, r.z};
      for (int i = 0; i < 3; ++i) {
        ManifoldRow row;
        row.valid = true;
        row.r = sw * rv[i];
        for (int j = 0; j < 6; ++j)
          row.J[j] = sw * ((J[3 * i] * dp[0][j] + J[3 * i + 1] * dp[1][j]) + J[3 * i + 2] * dp[2][j]);
        accumulate(ne, row);
        ++nr;
      }
    } else {
      ManifoldRow row;
      row.valid = true;
      row.r = sw * plane_residual(pw, c.normal, c.offset);
      for (int j = 0; j < 6; ++j)
        row.J[j] = sw * ((c.normal.x * dp[0][j] + c.normal.y * dp[1][j]) + c.normal.z * dp[2][j]);
      accumulate(ne, row);
      ++nr;
    }
  }
  if (rows) *rows = nr;
}

}  // namespace oracle
