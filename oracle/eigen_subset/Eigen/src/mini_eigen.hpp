// TEST INFRASTRUCTURE — a minimal, eagerly evaluated stand-in for the subset
// of Eigen 3 (MPL2; version unpinned by the reference, `>= 3.3` at
// proj/core/CMakeLists.txt:1, absent from this image) that the reference's
// hot-path sources use, so that those sources compile UNCHANGED from
// /root/reference into oracle/_ref/ (the reference arm / parity pin).
//
// Every expression is evaluated immediately into a plain matrix; views
// (block, row, col, head, segment, diagonal, transpose, Map) are strided
// pointers into existing storage. Sums run in ascending index order with
// plain multiply/add (the reference builds without -march, so Eigen's SSE2
// packets round like scalar code for the fixed-size 2/3-vectors it uses; its
// blocked GEMM/GEMV order is NOT reproduced — those results are compared
// with tolerances, SURVEY §8c "Eigen GEMM/LDLT bit patterns unpinned").
//
// Algorithms restated from Eigen's published sources (named per class):
//   LDLT                     — ldlt_inplace<Lower>::unblocked + LDLT::_solve_impl
//   SelfAdjointEigenSolver   — scale to [-1,1], tridiagonalization_inplace (3x3
//                              closed form / Householder), computeFromTridiagonal_impl
//                              with tridiagonal_qr_step (Wilkinson shift) and
//                              JacobiRotation::makeGivens, ascending sort
//   JacobiSVD (3x3)          — two-sided Jacobi (real 2x2 SVD per pair)
//   AngleAxis / Quaternion / Transform<Isometry> — toRotationMatrix,
//                              quaternion product, translate/rotate on the right
#pragma once

#include <algorithm>
#include <array>
#include <cassert>
#include <cmath>
#include <cstddef>
#include <initializer_list>
#include <limits>
#include <stdexcept>
#include <thread>
#include <type_traits>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
inline constexpr int Dynamic = -1;
enum StorageOptions { ColMajor = 0, RowMajor = 1, AutoAlign = 0, DontAlign = 2 };
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };
enum DecompositionOptions {
  ComputeEigenvectors = 0x80,
  EigenvaluesOnly = 0x40,
  ComputeFullU = 0x04,
  ComputeThinU = 0x08,
  ComputeFullV = 0x10,
  ComputeThinV = 0x20
};
enum UpLoType { Lower = 1, Upper = 2 };
enum TransformTraits { Isometry = 1, Affine = 2, AffineCompact = 3, Projective = 4 };

namespace internal {
constexpr int pick(int a, int b) { return a != Dynamic ? a : b; }
constexpr int mul_sz(int a, int b) { return (a == Dynamic || b == Dynamic) ? Dynamic : a * b; }
constexpr int min_sz(int a, int b) {
  return (a == Dynamic || b == Dynamic) ? Dynamic : (a < b ? a : b);
}
}  // namespace internal

template <int R, int C, bool A>
class Plain;
template <int R, int C, bool A>
class View;

struct DenseTag {};

template <class T>
inline constexpr bool is_dense_v = std::is_base_of_v<DenseTag, std::decay_t<T>>;
template <class T>
concept DenseExpr = is_dense_v<T>;

// ---------------------------------------------------------------------------
// CRTP base: everything is memory-backed (ptr + row/col strides).
template <class D, int R, int C, bool A>
class DenseBase : public DenseTag {
 public:
  static constexpr int RowsAtCompileTime = R;
  static constexpr int ColsAtCompileTime = C;
  static constexpr int SizeAtCompileTime = internal::mul_sz(R, C);
  static constexpr bool IsArray = A;
  static constexpr bool IsVectorAtCompileTime = (R == 1 || C == 1);
  using Scalar = double;
  using RealScalar = double;
  using PlainType = Plain<R, C, A>;

  D& derived() { return static_cast<D&>(*this); }
  const D& derived() const { return static_cast<const D&>(*this); }
  Index rows() const { return derived().rows(); }
  Index cols() const { return derived().cols(); }
  Index size() const { return rows() * cols(); }
  double* p() const { return derived().ptr(); }
  Index rstr() const { return derived().rs(); }
  Index cstr() const { return derived().cs(); }

  double coeff(Index i, Index j) const { return p()[i * rstr() + j * cstr()]; }
  double& coeffRef(Index i, Index j) const { return p()[i * rstr() + j * cstr()]; }
  // linear (vector) index; for matrices column-major order
  double& lin(Index k) const {
    if (rows() == 1) return coeffRef(0, k);
    if (cols() == 1) return coeffRef(k, 0);
    return coeffRef(k % rows(), k / rows());
  }
  double coeff(Index k) const { return lin(k); }
  double value() const { return coeff(0, 0); }
  double& coeffRef(Index k) const { return lin(k); }
  double& operator()(Index i, Index j) const { return coeffRef(i, j); }
  double& operator()(Index k) const { return lin(k); }
  double& operator[](Index k) const { return lin(k); }
  double& x() const { return lin(0); }
  double& y() const { return lin(1); }
  double& z() const { return lin(2); }
  double& w() const { return lin(3); }

  // ---- views ---------------------------------------------------------------
  template <int RR, int CC>
  View<RR, CC, A> view(Index i, Index j, Index r, Index c) const {
    return View<RR, CC, A>(p() + i * rstr() + j * cstr(), r, c, rstr(), cstr());
  }
  View<Dynamic, Dynamic, A> block(Index i, Index j, Index r, Index c) const {
    return view<Dynamic, Dynamic>(i, j, r, c);
  }
  template <int RR, int CC>
  View<RR, CC, A> block(Index i, Index j) const { return view<RR, CC>(i, j, RR, CC); }
  View<1, C, A> row(Index i) const { return view<1, C>(i, 0, 1, cols()); }
  View<R, 1, A> col(Index j) const { return view<R, 1>(0, j, rows(), 1); }
  View<R, Dynamic, A> middleCols(Index j, Index n) const { return view<R, Dynamic>(0, j, rows(), n); }
  template <int N>
  View<R, N, A> middleCols(Index j) const { return view<R, N>(0, j, rows(), N); }
  View<Dynamic, C, A> middleRows(Index i, Index n) const { return view<Dynamic, C>(i, 0, n, cols()); }
  template <int N>
  View<N, C, A> middleRows(Index i) const { return view<N, C>(i, 0, N, cols()); }
  View<R, Dynamic, A> leftCols(Index n) const { return view<R, Dynamic>(0, 0, rows(), n); }
  template <int N>
  View<R, N, A> leftCols() const { return view<R, N>(0, 0, rows(), N); }
  View<R, Dynamic, A> rightCols(Index n) const { return view<R, Dynamic>(0, cols() - n, rows(), n); }
  template <int N>
  View<R, N, A> rightCols() const { return view<R, N>(0, cols() - N, rows(), N); }
  View<Dynamic, C, A> topRows(Index n) const { return view<Dynamic, C>(0, 0, n, cols()); }
  template <int N>
  View<N, C, A> topRows() const { return view<N, C>(0, 0, N, cols()); }
  View<Dynamic, C, A> bottomRows(Index n) const { return view<Dynamic, C>(rows() - n, 0, n, cols()); }
  template <int N>
  View<N, C, A> bottomRows() const { return view<N, C>(rows() - N, 0, N, cols()); }
  View<Dynamic, Dynamic, A> topLeftCorner(Index r, Index c) const { return block(0, 0, r, c); }
  View<Dynamic, Dynamic, A> bottomRightCorner(Index r, Index c) const {
    return block(rows() - r, cols() - c, r, c);
  }
  // vector segments (row or column vectors)
  template <int N>
  auto head() const { return seg<N>(0, N); }
  template <int N>
  auto tail() const { return seg<N>(size() - N, N); }
  template <int N>
  auto segment(Index i) const { return seg<N>(i, N); }
  auto head(Index n) const { return seg<Dynamic>(0, n); }
  auto tail(Index n) const { return seg<Dynamic>(size() - n, n); }
  auto segment(Index i, Index n) const { return seg<Dynamic>(i, n); }
  template <int N>
  auto seg(Index i, Index n) const {
    if constexpr (R == 1)
      return view<1, N>(0, i, 1, n);
    else {
      assert(cols() == 1);
      return view<N, 1>(i, 0, n, 1);
    }
  }
  View<C, R, A> transpose() const { return View<C, R, A>(p(), cols(), rows(), cstr(), rstr()); }
  View<C, R, A> adjoint() const { return transpose(); }
  View<internal::min_sz(R, C), 1, A> diagonal() const {
    return View<internal::min_sz(R, C), 1, A>(p(), std::min(rows(), cols()), 1, rstr() + cstr(), 0);
  }
  View<R, C, true> array() const { return View<R, C, true>(p(), rows(), cols(), rstr(), cstr()); }
  View<R, C, false> matrix() const { return View<R, C, false>(p(), rows(), cols(), rstr(), cstr()); }
  D& noalias() { return derived(); }
  Plain<R, C, A> eval() const { return Plain<R, C, A>(derived()); }

  // ---- in-place ------------------------------------------------------------
  D& setZero() { return setConstant(0.0); }
  D& setOnes() { return setConstant(1.0); }
  D& setConstant(double v) {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) coeffRef(i, j) = v;
    return derived();
  }
  void fill(double v) { setConstant(v); }
  D& setIdentity() {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) coeffRef(i, j) = (i == j) ? 1.0 : 0.0;
    return derived();
  }
  template <DenseExpr E>
  void assign_from(const E& e) {
    // evaluate first (views may alias), then copy
    const Plain<E::RowsAtCompileTime, E::ColsAtCompileTime, E::IsArray> t(e);
    if (t.rows() != rows() || t.cols() != cols()) throw std::logic_error("mini-eigen: size mismatch");
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) coeffRef(i, j) = t.coeff(i, j);
  }
  template <DenseExpr E>
  D& operator+=(const E& e) {
    const Plain<E::RowsAtCompileTime, E::ColsAtCompileTime, E::IsArray> t(e);
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) coeffRef(i, j) = coeff(i, j) + t.coeff(i, j);
    return derived();
  }
  template <DenseExpr E>
  D& operator-=(const E& e) {
    const Plain<E::RowsAtCompileTime, E::ColsAtCompileTime, E::IsArray> t(e);
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) coeffRef(i, j) = coeff(i, j) - t.coeff(i, j);
    return derived();
  }
  template <DenseExpr E>
  D& operator*=(const E& e) {
    derived() = derived() * e;
    return derived();
  }
  D& operator*=(double s) {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) coeffRef(i, j) = coeff(i, j) * s;
    return derived();
  }
  D& operator/=(double s) {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) coeffRef(i, j) = coeff(i, j) / s;
    return derived();
  }
  // array-only scalar shifts
  D& operator+=(double s) requires A {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) coeffRef(i, j) = coeff(i, j) + s;
    return derived();
  }
  D& operator-=(double s) requires A {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) coeffRef(i, j) = coeff(i, j) - s;
    return derived();
  }
  template <DenseExpr E>
  void swap(const E& o) {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) std::swap(coeffRef(i, j), o.coeffRef(i, j));
  }
  void normalize() {
    const double n = norm();
    if (n > 0.0) *this /= n;
  }

  // ---- reductions ----------------------------------------------------------
  template <class F>
  Plain<R, C, A> unary(F f) const {
    Plain<R, C, A> out(rows(), cols());
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) out.coeffRef(i, j) = f(coeff(i, j));
    return out;
  }
  double sum() const {
    double s = 0.0;
    bool first = true;
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) {
        s = first ? coeff(i, j) : s + coeff(i, j);
        first = false;
      }
    return s;
  }
  double prod() const {
    double s = 1.0;
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) s *= coeff(i, j);
    return s;
  }
  double mean() const { return sum() / static_cast<double>(size()); }
  double squaredNorm() const {
    double s = 0.0;
    bool first = true;
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) {
        const double v = coeff(i, j) * coeff(i, j);
        s = first ? v : s + v;
        first = false;
      }
    return s;
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  Plain<R, C, A> normalized() const {
    const double n = norm();
    Plain<R, C, A> out(derived());
    if (n > 0.0) out /= n;
    return out;
  }
  double trace() const {
    double s = 0.0;
    for (Index i = 0; i < std::min(rows(), cols()); ++i) s = (i == 0) ? coeff(0, 0) : s + coeff(i, i);
    return s;
  }
  template <DenseExpr E>
  double dot(const E& o) const {
    double s = 0.0;
    for (Index k = 0; k < size(); ++k) s = (k == 0) ? lin(k) * o.lin(k) : s + lin(k) * o.lin(k);
    return s;
  }
  template <DenseExpr E>
  Plain<3, 1, A> cross(const E& o) const {
    Plain<3, 1, A> r;
    r(0) = lin(1) * o.lin(2) - lin(2) * o.lin(1);
    r(1) = lin(2) * o.lin(0) - lin(0) * o.lin(2);
    r(2) = lin(0) * o.lin(1) - lin(1) * o.lin(0);
    return r;
  }
  double maxCoeff() const {
    double m = coeff(0, 0);
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) m = std::max(m, coeff(i, j));
    return m;
  }
  double minCoeff() const {
    double m = coeff(0, 0);
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) m = std::min(m, coeff(i, j));
    return m;
  }
  // first index of the extremum in linear (column-major) order, as Eigen
  template <class I>
  double maxCoeff(I* idx) const {
    Index best = 0;
    for (Index k = 1; k < size(); ++k)
      if (lin(k) > lin(best)) best = k;
    *idx = static_cast<I>(best);
    return lin(best);
  }
  template <class I>
  double minCoeff(I* idx) const {
    Index best = 0;
    for (Index k = 1; k < size(); ++k)
      if (lin(k) < lin(best)) best = k;
    *idx = static_cast<I>(best);
    return lin(best);
  }
  bool allFinite() const {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i)
        if (!std::isfinite(coeff(i, j))) return false;
    return true;
  }
  bool hasNaN() const {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i)
        if (std::isnan(coeff(i, j))) return true;
    return false;
  }
  bool all() const {
    for (Index k = 0; k < size(); ++k)
      if (lin(k) == 0.0) return false;
    return true;
  }
  bool any() const {
    for (Index k = 0; k < size(); ++k)
      if (lin(k) != 0.0) return true;
    return false;
  }
  Index count() const {
    Index n = 0;
    for (Index k = 0; k < size(); ++k) n += (lin(k) != 0.0);
    return n;
  }
  template <DenseExpr E>
  bool isApprox(const E& o, double prec = 1e-12) const {
    const Plain<R, C, false> d = (derived().matrix() - o.matrix());
    return d.norm() <= prec * std::min(norm(), o.norm());
  }
  bool isZero(double prec = 1e-12) const {
    for (Index k = 0; k < size(); ++k)
      if (std::abs(lin(k)) > prec) return false;
    return true;
  }
  Plain<R, C, A> cwiseAbs() const { return unary([](double v) { return std::abs(v); }); }
  Plain<R, C, A> cwiseAbs2() const { return unary([](double v) { return v * v; }); }
  Plain<R, C, A> cwiseSqrt() const { return unary([](double v) { return std::sqrt(v); }); }
  Plain<R, C, A> cwiseInverse() const { return unary([](double v) { return 1.0 / v; }); }
  Plain<R, C, A> cwiseMax(double s) const { return unary([s](double v) { return std::max(v, s); }); }
  Plain<R, C, A> cwiseMin(double s) const { return unary([s](double v) { return std::min(v, s); }); }
  template <DenseExpr E>
  Plain<R, C, A> cwiseMax(const E& o) const { return binary(o, [](double a, double b) { return std::max(a, b); }); }
  template <DenseExpr E>
  Plain<R, C, A> cwiseMin(const E& o) const { return binary(o, [](double a, double b) { return std::min(a, b); }); }
  template <DenseExpr E>
  Plain<R, C, A> cwiseProduct(const E& o) const { return binary(o, [](double a, double b) { return a * b; }); }
  template <DenseExpr E>
  Plain<R, C, A> cwiseQuotient(const E& o) const { return binary(o, [](double a, double b) { return a / b; }); }
  template <DenseExpr E, class F>
  Plain<R, C, A> binary(const E& o, F f) const {
    Plain<R, C, A> out(rows(), cols());
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) out.coeffRef(i, j) = f(coeff(i, j), o.coeff(i, j));
    return out;
  }
  // array functions
  Plain<R, C, A> abs() const { return cwiseAbs(); }
  Plain<R, C, A> sqrt() const { return cwiseSqrt(); }
  Plain<R, C, A> square() const { return cwiseAbs2(); }
  Plain<R, C, A> exp() const { return unary([](double v) { return std::exp(v); }); }
  Plain<R, C, A> max(double s) const { return cwiseMax(s); }
  Plain<R, C, A> min(double s) const { return cwiseMin(s); }
  template <DenseExpr E>
  Plain<R, C, A> max(const E& o) const { return cwiseMax(o); }
  template <DenseExpr E>
  Plain<R, C, A> min(const E& o) const { return cwiseMin(o); }

  // ---- small dense algebra -------------------------------------------------
  double determinant() const;
  Plain<R, C, false> inverse() const;
  auto ldlt() const;
  auto llt() const;
  template <int UpLo>
  auto selfadjointView() const { return derived(); }
  auto asDiagonal() const;
};

// ---------------------------------------------------------------------------
template <int R, int C, bool A>
class Plain : public DenseBase<Plain<R, C, A>, R, C, A> {
  using Base = DenseBase<Plain<R, C, A>, R, C, A>;
  static constexpr bool kFixed = (R != Dynamic && C != Dynamic);
  using Store = std::conditional_t<kFixed, std::array<double, (kFixed ? R * C : 1)>, std::vector<double>>;
  Store d_{};
  Index r_ = (R == Dynamic ? 0 : R), c_ = (C == Dynamic ? 0 : C);

 public:
  using Base::operator+=;
  using Base::operator-=;
  using Base::operator*=;
  using Base::operator/=;

  Plain() { zero_init(); }
  // Dynamic vectors: Plain(n); dynamic matrices: Plain(r, c)
  explicit Plain(Index n) requires(!kFixed && (R == 1 || C == 1)) {
    resize(R == 1 ? 1 : n, R == 1 ? n : 1);
  }
  explicit Plain(int n) requires(!kFixed && (R == 1 || C == 1)) : Plain(static_cast<Index>(n)) {}
  Plain(Index r, Index c) requires(!kFixed) { resize(r, c); }
  Plain(int r, int c) requires(!kFixed) { resize(r, c); }
  Plain(Index r, long c) requires(!kFixed && !std::is_same_v<long, Index>) { resize(r, c); }
  // fixed small vectors: coefficients
  Plain(double a, double b) requires(kFixed && R * C == 2) {
    d_[0] = a;
    d_[1] = b;
  }
  Plain(double a, double b, double c) requires(kFixed && R * C == 3) {
    d_[0] = a;
    d_[1] = b;
    d_[2] = c;
  }
  Plain(double a, double b, double c, double e) requires(kFixed && R * C == 4 && (R == 1 || C == 1)) {
    d_[0] = a;
    d_[1] = b;
    d_[2] = c;
    d_[3] = e;
  }
  // Fixed shape constructed with explicit (rows, cols) equal to its shape.
  Plain(Index r, Index c) requires(kFixed && !(R * C == 2)) {
    if (r != R || c != C) throw std::logic_error("mini-eigen: fixed size mismatch");
  }
  Plain(const Plain&) = default;
  Plain(Plain&&) = default;
  template <DenseExpr E>
  Plain(const E& e) {
    resize(e.rows(), e.cols());
    for (Index j = 0; j < e.cols(); ++j)
      for (Index i = 0; i < e.rows(); ++i) coeffRef(i, j) = e.coeff(i, j);
  }
  Plain& operator=(const Plain& o) {
    if (this != &o) {
      resize(o.rows(), o.cols());
      d_ = o.d_;
    }
    return *this;
  }
  Plain& operator=(Plain&& o) {
    if constexpr (kFixed)
      d_ = o.d_;
    else {
      d_ = std::move(o.d_);
      r_ = o.r_;
      c_ = o.c_;
    }
    return *this;
  }
  template <DenseExpr E>
  Plain& operator=(const E& e) {
    const Plain<E::RowsAtCompileTime, E::ColsAtCompileTime, E::IsArray> t(e);
    resize(t.rows(), t.cols());
    for (Index j = 0; j < t.cols(); ++j)
      for (Index i = 0; i < t.rows(); ++i) coeffRef(i, j) = t.coeff(i, j);
    return *this;
  }

  Index rows() const { return r_; }
  Index cols() const { return c_; }
  double* ptr() const { return const_cast<double*>(d_.data()); }
  Index rs() const { return 1; }
  Index cs() const { return r_; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  using Base::coeff;
  using Base::coeffRef;

  void zero_init() {
    if constexpr (kFixed) d_.fill(0.0);
  }
  void resize(Index r, Index c) {
    if constexpr (kFixed) {
      if (r != R || c != C) throw std::logic_error("mini-eigen: cannot resize a fixed-size matrix");
    } else {
      if (R != Dynamic && r != R) throw std::logic_error("mini-eigen: row count is fixed");
      if (C != Dynamic && c != C) throw std::logic_error("mini-eigen: column count is fixed");
      r_ = r;
      c_ = c;
      d_.assign(static_cast<std::size_t>(r * c), 0.0);
    }
  }
  void resize(Index n) {
    if (R == 1)
      resize(1, n);
    else
      resize(n, 1);
  }
  void conservativeResize(Index r, Index c) {
    Plain old(*this);
    resize(r, c);
    for (Index j = 0; j < std::min(c, old.cols()); ++j)
      for (Index i = 0; i < std::min(r, old.rows()); ++i) coeffRef(i, j) = old.coeff(i, j);
  }
  void conservativeResize(Index n) {
    if (R == 1)
      conservativeResize(1, n);
    else
      conservativeResize(n, 1);
  }
  Plain& setZero(Index n) {
    resize(n);
    return *this;
  }
  Plain& setZero(Index r, Index c) {
    resize(r, c);
    return *this;
  }
  Plain& setOnes(Index r, Index c) {
    resize(r, c);
    this->setConstant(1.0);
    return *this;
  }
  using Base::setOnes;
  using Base::setZero;

  static Plain Zero() { return Plain(); }
  static Plain Zero(Index n) { return Plain(n); }
  static Plain Zero(Index r, Index c) { return Plain(r, c); }
  static Plain Ones() { return Constant(1.0); }
  static Plain Ones(Index n) { return Constant(n, 1.0); }
  static Plain Ones(Index r, Index c) { return Constant(r, c, 1.0); }
  static Plain Constant(double v) {
    Plain m;
    m.setConstant(v);
    return m;
  }
  static Plain Constant(Index n, double v) {
    Plain m(n);
    m.setConstant(v);
    return m;
  }
  static Plain Constant(Index r, Index c, double v) {
    Plain m(r, c);
    m.setConstant(v);
    return m;
  }
  static Plain Identity() {
    Plain m;
    m.setIdentity();
    return m;
  }
  static Plain Identity(Index r, Index c) {
    Plain m(r, c);
    m.setIdentity();
    return m;
  }
  static Plain Unit(Index i) {
    Plain m;
    m(i) = 1.0;
    return m;
  }
  static Plain UnitX() { return Unit(0); }
  static Plain UnitY() { return Unit(1); }
  static Plain UnitZ() { return Unit(2); }

  // comma initializer (row-major fill, as Eigen's)
  struct Comma {
    Plain& m;
    Index k;
    Comma& operator,(double v) {
      m.coeffRef(k / m.cols(), k % m.cols()) = v;
      ++k;
      return *this;
    }
  };
  Comma operator<<(double v) {
    this->coeffRef(0, 0) = v;
    return Comma{*this, 1};
  }
};

// ---------------------------------------------------------------------------
template <int R, int C, bool A>
class View : public DenseBase<View<R, C, A>, R, C, A> {
  using Base = DenseBase<View<R, C, A>, R, C, A>;
  double* p_;
  Index r_, c_, rs_, cs_;

 public:
  View(double* p, Index r, Index c, Index rs, Index cs) : p_(p), r_(r), c_(c), rs_(rs), cs_(cs) {}
  View(const View&) = default;
  View& operator=(const View& o) {
    this->assign_from(o);
    return *this;
  }
  template <DenseExpr E>
  View& operator=(const E& e) {
    this->assign_from(e);
    return *this;
  }
  using Base::operator+=;
  using Base::operator-=;
  using Base::operator*=;
  using Base::operator/=;
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  double* ptr() const { return p_; }
  Index rs() const { return rs_; }
  Index cs() const { return cs_; }
  double* data() const { return p_; }
  // comma initializer into a view
  struct Comma {
    const View& m;
    Index k;
    Comma& operator,(double v) {
      m.coeffRef(k / m.cols(), k % m.cols()) = v;
      ++k;
      return *this;
    }
  };
  Comma operator<<(double v) const {
    this->coeffRef(0, 0) = v;
    return Comma{*this, 1};
  }
};

template <class S, int R, int C, int Opt = 0, int MR = R, int MC = C>
using Matrix = Plain<R, C, false>;
template <class S, int R, int C, int Opt = 0, int MR = R, int MC = C>
using Array = Plain<R, C, true>;

using MatrixXd = Plain<Dynamic, Dynamic, false>;
using VectorXd = Plain<Dynamic, 1, false>;
using RowVectorXd = Plain<1, Dynamic, false>;
using Vector2d = Plain<2, 1, false>;
using Vector3d = Plain<3, 1, false>;
using Vector4d = Plain<4, 1, false>;
using Vector6d = Plain<6, 1, false>;
using RowVector2d = Plain<1, 2, false>;
using RowVector3d = Plain<1, 3, false>;
using Matrix2d = Plain<2, 2, false>;
using Matrix3d = Plain<3, 3, false>;
using Matrix4d = Plain<4, 4, false>;
using ArrayXd = Plain<Dynamic, 1, true>;
using Array3d = Plain<3, 1, true>;
using Array2d = Plain<2, 1, true>;

// Map<const VectorXd>(ptr, n) / Map<MatrixXd>(ptr, r, c): column-major view
template <class M>
class Map : public View<std::remove_const_t<M>::RowsAtCompileTime, std::remove_const_t<M>::ColsAtCompileTime,
                        std::remove_const_t<M>::IsArray> {
  using P = std::remove_const_t<M>;
  using V = View<P::RowsAtCompileTime, P::ColsAtCompileTime, P::IsArray>;
  using Ptr = std::conditional_t<std::is_const_v<M>, const double*, double*>;

 public:
  Map(Ptr p, Index n)
      : V(const_cast<double*>(p), P::RowsAtCompileTime == 1 ? 1 : n, P::RowsAtCompileTime == 1 ? n : 1, 1,
          P::RowsAtCompileTime == 1 ? 1 : n) {}
  Map(Ptr p, Index r, Index c) : V(const_cast<double*>(p), r, c, 1, r) {}
  explicit Map(Ptr p) : V(const_cast<double*>(p), P::RowsAtCompileTime, P::ColsAtCompileTime, 1,
                          P::RowsAtCompileTime) {}
  using V::operator=;
};

// ---------------------------------------------------------------------------
// arithmetic (eager)
namespace internal {
template <class X, class Y>
using sum_t = Plain<pick(X::RowsAtCompileTime, Y::RowsAtCompileTime),
                    pick(X::ColsAtCompileTime, Y::ColsAtCompileTime), X::IsArray>;
template <class X, class Y>
using prod_t = Plain<X::RowsAtCompileTime, Y::ColsAtCompileTime, false>;
template <class X>
using plain_t = Plain<X::RowsAtCompileTime, X::ColsAtCompileTime, X::IsArray>;

inline void check_same(Index r1, Index c1, Index r2, Index c2) {
  if (r1 != r2 || c1 != c2) throw std::logic_error("mini-eigen: operand sizes differ");
}
}  // namespace internal

template <DenseExpr X, DenseExpr Y>
auto operator+(const X& a, const Y& b) {
  internal::check_same(a.rows(), a.cols(), b.rows(), b.cols());
  internal::sum_t<X, Y> out(a);
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) out.coeffRef(i, j) = a.coeff(i, j) + b.coeff(i, j);
  return out;
}
template <DenseExpr X, DenseExpr Y>
auto operator-(const X& a, const Y& b) {
  internal::check_same(a.rows(), a.cols(), b.rows(), b.cols());
  internal::sum_t<X, Y> out(a);
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) out.coeffRef(i, j) = a.coeff(i, j) - b.coeff(i, j);
  return out;
}
template <DenseExpr X>
auto operator-(const X& a) {
  return a.unary([](double v) { return -v; });
}
template <DenseExpr X>
auto operator*(const X& a, double s) {
  return a.unary([s](double v) { return v * s; });
}
template <DenseExpr X>
auto operator*(double s, const X& a) {
  return a.unary([s](double v) { return s * v; });
}
template <DenseExpr X>
auto operator/(const X& a, double s) {
  return a.unary([s](double v) { return v / s; });
}
template <DenseExpr X>
  requires X::IsArray
auto operator+(const X& a, double s) {
  return a.unary([s](double v) { return v + s; });
}
template <DenseExpr X>
  requires X::IsArray
auto operator-(const X& a, double s) {
  return a.unary([s](double v) { return v - s; });
}
template <DenseExpr X>
  requires X::IsArray
auto operator+(double s, const X& a) {
  return a.unary([s](double v) { return s + v; });
}
template <DenseExpr X>
  requires X::IsArray
auto operator-(double s, const X& a) {
  return a.unary([s](double v) { return s - v; });
}
template <DenseExpr X, DenseExpr Y>
  requires(X::IsArray && Y::IsArray)
auto operator/(const X& a, const Y& b) {
  return a.cwiseQuotient(b);
}

// Matrix product: entry (i, j) = a(i,0) b(0,j) + a(i,1) b(1,j) + ..., k
// ascending, for every shape (so the result does not depend on the layout
// path taken or on the thread count). Column-major left operands run as
// column axpys (vectorisable without reassociation), transposed ones as
// contiguous dots; large products split output columns (or, for one column,
// rows) over std::thread workers — test-infrastructure speed only.
namespace internal {
inline unsigned product_threads(double work) {
  if (work < 4e6) return 1;
  const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
  return static_cast<unsigned>(std::min<double>(hc, std::max(1.0, work / 2e6)));
}
template <class F>
void parallel_range(Index n, unsigned threads, F f) {
  if (threads <= 1 || n < 2) {
    f(Index(0), n);
    return;
  }
  threads = static_cast<unsigned>(std::min<Index>(threads, n));
  std::vector<std::thread> pool;
  const Index chunk = (n + threads - 1) / threads;
  for (unsigned w = 0; w < threads; ++w) {
    const Index b = w * chunk, e = std::min(n, b + chunk);
    if (b < e) pool.emplace_back(f, b, e);
  }
  for (auto& t : pool) t.join();
}
}  // namespace internal

template <DenseExpr X, DenseExpr Y>
auto operator*(const X& a, const Y& b) {
  if constexpr (X::IsArray && Y::IsArray) {
    return a.cwiseProduct(b);
  } else {
    if (a.cols() != b.rows()) throw std::logic_error("mini-eigen: product size mismatch");
    internal::prod_t<X, Y> out(a.rows(), b.cols());
    const Index n = a.rows(), m = b.cols(), kk = a.cols();
    if (n == 0 || m == 0 || kk == 0) return out;
    const double* ap = a.p();
    const Index ars = a.rstr(), acs = a.cstr();
    const double* bp = b.p();
    const Index brs = b.rstr(), bcs = b.cstr();
    double* op = out.data();  // column-major, ld = n
    const unsigned th = internal::product_threads(double(n) * double(m) * double(kk));
    if (ars == 1) {
      auto cols = [&](Index j0, Index j1, Index i0, Index i1) {
        for (Index j = j0; j < j1; ++j) {
          double* oc = op + j * n;
          for (Index k = 0; k < kk; ++k) {
            const double bkj = bp[k * brs + j * bcs];
            const double* ac = ap + k * acs;
            if (k == 0)
              for (Index i = i0; i < i1; ++i) oc[i] = ac[i] * bkj;
            else
              for (Index i = i0; i < i1; ++i) oc[i] += ac[i] * bkj;
          }
        }
      };
      if (m == 1)
        internal::parallel_range(n, th, [&](Index i0, Index i1) { cols(0, 1, i0, i1); });
      else
        internal::parallel_range(m, th, [&](Index j0, Index j1) { cols(j0, j1, 0, n); });
    } else {
      auto rows = [&](Index j0, Index j1, Index i0, Index i1) {
        for (Index j = j0; j < j1; ++j)
          for (Index i = i0; i < i1; ++i) {
            const double* ar = ap + i * ars;
            const double* bc = bp + j * bcs;
            double s = ar[0] * bc[0];
            for (Index k = 1; k < kk; ++k) s += ar[k * acs] * bc[k * brs];
            op[i + j * n] = s;
          }
      };
      if (m == 1)
        internal::parallel_range(n, th, [&](Index i0, Index i1) { rows(0, 1, i0, i1); });
      else
        internal::parallel_range(m, th, [&](Index j0, Index j1) { rows(j0, j1, 0, n); });
    }
    return out;
  }
}

// 1x1 products convert to scalars through value()
template <DenseExpr X>
double value_of(const X& x) {
  return x.coeff(0, 0);
}

// ---------------------------------------------------------------------------
// small dense algebra
template <class D, int R, int C, bool A>
double DenseBase<D, R, C, A>::determinant() const {
  const Index n = rows();
  if (n == 1) return coeff(0, 0);
  if (n == 2) return coeff(0, 0) * coeff(1, 1) - coeff(0, 1) * coeff(1, 0);
  if (n == 3)
    return coeff(0, 0) * (coeff(1, 1) * coeff(2, 2) - coeff(2, 1) * coeff(1, 2)) -
           coeff(1, 0) * (coeff(0, 1) * coeff(2, 2) - coeff(2, 1) * coeff(0, 2)) +
           coeff(2, 0) * (coeff(0, 1) * coeff(1, 2) - coeff(1, 1) * coeff(0, 2));
  // partial-pivot LU
  Plain<Dynamic, Dynamic, false> m(derived());
  double det = 1.0;
  for (Index k = 0; k < n; ++k) {
    Index piv = k;
    for (Index i = k + 1; i < n; ++i)
      if (std::abs(m(i, k)) > std::abs(m(piv, k))) piv = i;
    if (m(piv, k) == 0.0) return 0.0;
    if (piv != k) {
      m.row(k).swap(m.row(piv));
      det = -det;
    }
    det *= m(k, k);
    for (Index i = k + 1; i < n; ++i) {
      const double f = m(i, k) / m(k, k);
      for (Index j = k; j < n; ++j) m(i, j) -= f * m(k, j);
    }
  }
  return det;
}

template <class D, int R, int C, bool A>
Plain<R, C, false> DenseBase<D, R, C, A>::inverse() const {
  const Index n = rows();
  Plain<R, C, false> out(derived());
  if (n == 2) {
    const double det = determinant();
    out(0, 0) = coeff(1, 1) / det;
    out(1, 1) = coeff(0, 0) / det;
    out(0, 1) = -coeff(0, 1) / det;
    out(1, 0) = -coeff(1, 0) / det;
    return out;
  }
  if (n == 3) {
    // cofactors / determinant (Eigen's compute_inverse_size3)
    const double c00 = coeff(1, 1) * coeff(2, 2) - coeff(1, 2) * coeff(2, 1);
    const double c10 = coeff(0, 2) * coeff(2, 1) - coeff(0, 1) * coeff(2, 2);
    const double c20 = coeff(0, 1) * coeff(1, 2) - coeff(0, 2) * coeff(1, 1);
    const double det = coeff(0, 0) * c00 + coeff(1, 0) * c10 + coeff(2, 0) * c20;
    out(0, 0) = c00 / det;
    out(0, 1) = c10 / det;
    out(0, 2) = c20 / det;
    out(1, 0) = (coeff(1, 2) * coeff(2, 0) - coeff(1, 0) * coeff(2, 2)) / det;
    out(1, 1) = (coeff(0, 0) * coeff(2, 2) - coeff(0, 2) * coeff(2, 0)) / det;
    out(1, 2) = (coeff(0, 2) * coeff(1, 0) - coeff(0, 0) * coeff(1, 2)) / det;
    out(2, 0) = (coeff(1, 0) * coeff(2, 1) - coeff(1, 1) * coeff(2, 0)) / det;
    out(2, 1) = (coeff(0, 1) * coeff(2, 0) - coeff(0, 0) * coeff(2, 1)) / det;
    out(2, 2) = (coeff(0, 0) * coeff(1, 1) - coeff(0, 1) * coeff(1, 0)) / det;
    return out;
  }
  // Gauss-Jordan with partial pivoting
  Plain<Dynamic, Dynamic, false> m(derived());
  Plain<Dynamic, Dynamic, false> inv = Plain<Dynamic, Dynamic, false>::Identity(n, n);
  for (Index k = 0; k < n; ++k) {
    Index piv = k;
    for (Index i = k + 1; i < n; ++i)
      if (std::abs(m(i, k)) > std::abs(m(piv, k))) piv = i;
    if (piv != k) {
      m.row(k).swap(m.row(piv));
      inv.row(k).swap(inv.row(piv));
    }
    const double d = m(k, k);
    for (Index j = 0; j < n; ++j) {
      m(k, j) /= d;
      inv(k, j) /= d;
    }
    for (Index i = 0; i < n; ++i)
      if (i != k) {
        const double f = m(i, k);
        for (Index j = 0; j < n; ++j) {
          m(i, j) -= f * m(k, j);
          inv(i, j) -= f * inv(k, j);
        }
      }
  }
  out = inv;
  return out;
}

// ---------------------------------------------------------------------------
// LDLT (Eigen/src/Cholesky/LDLT.h: ldlt_inplace<Lower>::unblocked, _solve_impl)
template <class MatrixType>
class LDLT {
 public:
  LDLT() = default;
  template <DenseExpr E>
  explicit LDLT(const E& a) {
    compute(a);
  }
  template <DenseExpr E>
  LDLT& compute(const E& a) {
    m_ = MatrixXd(a);
    const Index n = m_.rows();
    transp_.assign(static_cast<std::size_t>(n), 0);
    std::vector<double> temp(static_cast<std::size_t>(n), 0.0);
    enum { PositiveSemiDef = 1, NegativeSemiDef = 2, ZeroSign = 3, Indefinite = 4 };
    int sign = ZeroSign;
    bool ret = true, found_zero = false;
    for (Index k = 0; k < n; ++k) {
      // largest remaining diagonal entry (first on ties)
      Index big = k;
      double bv = std::abs(m_(k, k));
      for (Index i = k + 1; i < n; ++i)
        if (std::abs(m_(i, i)) > bv) {
          bv = std::abs(m_(i, i));
          big = i;
        }
      transp_[static_cast<std::size_t>(k)] = big;
      if (big != k) {
        for (Index c = 0; c < k; ++c) std::swap(m_(k, c), m_(big, c));
        for (Index r = big + 1; r < n; ++r) std::swap(m_(r, k), m_(r, big));
        std::swap(m_(k, k), m_(big, big));
        for (Index i = k + 1; i < big; ++i) {
          const double t = m_(i, k);
          m_(i, k) = m_(big, i);
          m_(big, i) = t;
        }
      }
      const Index rs = n - k - 1;
      if (k > 0) {
        for (Index c = 0; c < k; ++c) temp[static_cast<std::size_t>(c)] = m_(c, c) * m_(k, c);
        double s = 0.0;
        for (Index c = 0; c < k; ++c) s = (c == 0) ? m_(k, c) * temp[0] : s + m_(k, c) * temp[static_cast<std::size_t>(c)];
        m_(k, k) -= s;
        for (Index r = k + 1; r < n; ++r) {
          double acc = 0.0;
          for (Index c = 0; c < k; ++c) acc = (c == 0) ? m_(r, c) * temp[0] : acc + m_(r, c) * temp[static_cast<std::size_t>(c)];
          m_(r, k) -= acc;
        }
      }
      const double akk = m_(k, k);
      const bool valid = std::abs(akk) > 0.0;
      if (k == 0 && !valid) {
        sign = ZeroSign;
        for (Index j = 0; j < n; ++j) transp_[static_cast<std::size_t>(j)] = j;
        break;
      }
      if (rs > 0 && valid) {
        for (Index r = k + 1; r < n; ++r) m_(r, k) /= akk;
      } else if (rs > 0) {
        for (Index r = k + 1; r < n; ++r) ret = ret && (m_(r, k) == 0.0);
      }
      if (found_zero && valid)
        ret = false;
      else if (!valid)
        found_zero = true;
      if (sign == PositiveSemiDef) {
        if (akk < 0.0) sign = Indefinite;
      } else if (sign == NegativeSemiDef) {
        if (akk > 0.0) sign = Indefinite;
      } else if (sign == ZeroSign) {
        if (akk > 0.0)
          sign = PositiveSemiDef;
        else if (akk < 0.0)
          sign = NegativeSemiDef;
      }
    }
    positive_ = (sign == PositiveSemiDef || sign == ZeroSign);
    info_ = ret ? Success : NumericalIssue;
    return *this;
  }
  ComputationInfo info() const { return info_; }
  bool isPositive() const { return positive_; }
  bool isNegative() const { return !positive_; }
  VectorXd vectorD() const {
    VectorXd d(m_.rows());
    for (Index i = 0; i < m_.rows(); ++i) d(i) = m_(i, i);
    return d;
  }
  const MatrixXd& matrixLDLT() const { return m_; }
  template <DenseExpr E>
  Plain<E::RowsAtCompileTime, E::ColsAtCompileTime, false> solve(const E& b) const {
    Plain<E::RowsAtCompileTime, E::ColsAtCompileTime, false> x(b);
    const Index n = m_.rows(), nr = x.cols();
    // x = P b
    for (Index k = 0; k < n; ++k) {
      const Index t = transp_[static_cast<std::size_t>(k)];
      if (t != k)
        for (Index c = 0; c < nr; ++c) std::swap(x(k, c), x(t, c));
    }
    // L^-1 (unit lower, forward)
    for (Index c = 0; c < nr; ++c)
      for (Index i = 0; i < n; ++i) {
        const double xi = x(i, c);
        for (Index r = i + 1; r < n; ++r) x(r, c) -= m_(r, i) * xi;
      }
    // D^+ (pseudo-inverse below the smallest normal number)
    const double tol = std::numeric_limits<double>::min();
    for (Index i = 0; i < n; ++i) {
      const double d = m_(i, i);
      for (Index c = 0; c < nr; ++c) {
        if (std::abs(d) > tol)
          x(i, c) /= d;
        else
          x(i, c) = 0.0;
      }
    }
    // L^-T (backward)
    for (Index c = 0; c < nr; ++c)
      for (Index i = n - 1; i >= 0; --i) {
        double s = x(i, c);
        for (Index r = i + 1; r < n; ++r) s -= m_(r, i) * x(r, c);
        x(i, c) = s;
      }
    // P^T
    for (Index k = n - 1; k >= 0; --k) {
      const Index t = transp_[static_cast<std::size_t>(k)];
      if (t != k)
        for (Index c = 0; c < nr; ++c) std::swap(x(k, c), x(t, c));
    }
    return x;
  }

 private:
  MatrixXd m_;
  std::vector<Index> transp_;
  bool positive_ = true;
  ComputationInfo info_ = Success;
};

// LLT (plain Cholesky, lower)
template <class MatrixType>
class LLT {
 public:
  template <DenseExpr E>
  explicit LLT(const E& a) : l_(a) {
    const Index n = l_.rows();
    for (Index k = 0; k < n; ++k) {
      double d = l_(k, k);
      for (Index c = 0; c < k; ++c) d -= l_(k, c) * l_(k, c);
      if (!(d > 0.0)) {
        info_ = NumericalIssue;
        return;
      }
      d = std::sqrt(d);
      l_(k, k) = d;
      for (Index r = k + 1; r < n; ++r) {
        double s = l_(r, k);
        for (Index c = 0; c < k; ++c) s -= l_(r, c) * l_(k, c);
        l_(r, k) = s / d;
      }
    }
  }
  ComputationInfo info() const { return info_; }
  template <DenseExpr E>
  Plain<E::RowsAtCompileTime, E::ColsAtCompileTime, false> solve(const E& b) const {
    Plain<E::RowsAtCompileTime, E::ColsAtCompileTime, false> x(b);
    const Index n = l_.rows();
    for (Index c = 0; c < x.cols(); ++c) {
      for (Index i = 0; i < n; ++i) {
        double s = x(i, c);
        for (Index k = 0; k < i; ++k) s -= l_(i, k) * x(k, c);
        x(i, c) = s / l_(i, i);
      }
      for (Index i = n - 1; i >= 0; --i) {
        double s = x(i, c);
        for (Index k = i + 1; k < n; ++k) s -= l_(k, i) * x(k, c);
        x(i, c) = s / l_(i, i);
      }
    }
    return x;
  }

 private:
  MatrixXd l_;
  ComputationInfo info_ = Success;
};

template <class D, int R, int C, bool A>
auto DenseBase<D, R, C, A>::ldlt() const {
  return LDLT<Plain<R, C, false>>(derived());
}
template <class D, int R, int C, bool A>
auto DenseBase<D, R, C, A>::llt() const {
  return LLT<Plain<R, C, false>>(derived());
}
template <class D, int R, int C, bool A>
auto DenseBase<D, R, C, A>::asDiagonal() const {
  Plain<internal::pick(R, C) == 1 ? internal::pick(C, R) : internal::pick(R, C),
        internal::pick(R, C) == 1 ? internal::pick(C, R) : internal::pick(R, C), false>
      out(size(), size());
  out.setZero();
  for (Index i = 0; i < size(); ++i) out(i, i) = lin(i);
  return out;
}

// ---------------------------------------------------------------------------
// JacobiRotation::makeGivens (real) and the tridiagonal QR step
namespace internal {
struct Givens {
  double c = 1.0, s = 0.0;
  void make(double p, double q) {
    if (q == 0.0) {
      c = p < 0.0 ? -1.0 : 1.0;
      s = 0.0;
    } else if (p == 0.0) {
      c = 0.0;
      s = q < 0.0 ? 1.0 : -1.0;
    } else if (std::abs(p) > std::abs(q)) {
      const double t = q / p;
      double u = std::sqrt(1.0 + t * t);
      if (p < 0.0) u = -u;
      c = 1.0 / u;
      s = -t * c;
    } else {
      const double t = p / q;
      double u = std::sqrt(1.0 + t * t);
      if (q < 0.0) u = -u;
      s = -1.0 / u;
      c = -t * s;
    }
  }
};

// Q <- Q G on columns (k, k+1): x' = c x - s y, y' = s x + c y
inline void apply_right(MatrixXd& q, Index k, const Givens& g) {
  for (Index i = 0; i < q.rows(); ++i) {
    const double xi = q(i, k), yi = q(i, k + 1);
    q(i, k) = g.c * xi - g.s * yi;
    q(i, k + 1) = g.s * xi + g.c * yi;
  }
}

inline void tridiagonal_qr_step(double* diag, double* subdiag, Index start, Index end, MatrixXd* q) {
  const double td = (diag[end - 1] - diag[end]) * 0.5;
  const double e = subdiag[end - 1];
  double mu = diag[end];
  if (td == 0.0) {
    mu -= std::abs(e);
  } else if (e != 0.0) {
    const double e2 = e * e;
    const double h = std::hypot(td, e);
    if (e2 == 0.0)
      mu -= e / ((td + (td > 0.0 ? h : -h)) / e);
    else
      mu -= e2 / (td + (td > 0.0 ? h : -h));
  }
  double x = diag[start] - mu;
  double z = subdiag[start];
  for (Index k = start; k < end && z != 0.0; ++k) {
    Givens rot;
    rot.make(x, z);
    const double sdk = rot.s * diag[k] + rot.c * subdiag[k];
    const double dkp1 = rot.s * subdiag[k] + rot.c * diag[k + 1];
    diag[k] = rot.c * (rot.c * diag[k] - rot.s * subdiag[k]) - rot.s * (rot.c * subdiag[k] - rot.s * diag[k + 1]);
    diag[k + 1] = rot.s * sdk + rot.c * dkp1;
    subdiag[k] = rot.c * sdk - rot.s * dkp1;
    if (k > start) subdiag[k - 1] = rot.c * subdiag[k - 1] - rot.s * z;
    x = subdiag[k];
    if (k < end - 1) {
      z = -rot.s * subdiag[k + 1];
      subdiag[k + 1] = rot.c * subdiag[k + 1];
    }
    if (q) apply_right(*q, k, rot);
  }
}
}  // namespace internal

template <class MatrixType>
class SelfAdjointEigenSolver {
 public:
  using EV = Plain<MatrixType::RowsAtCompileTime, 1, false>;
  SelfAdjointEigenSolver() = default;
  template <DenseExpr E>
  explicit SelfAdjointEigenSolver(const E& a, int options = ComputeEigenvectors) {
    compute(a, options);
  }
  template <DenseExpr E>
  SelfAdjointEigenSolver& compute(const E& a, int options = ComputeEigenvectors) {
    const bool vecs = (options & ComputeEigenvectors) == ComputeEigenvectors;
    const Index n = a.cols();
    MatrixXd mat(n, n);
    VectorXd diag(n);
    if (n == 1) {
      diag(0) = a.coeff(0, 0);
      mat(0, 0) = 1.0;
      eivalues_ = diag;
      eivec_ = mat;
      info_ = Success;
      return *this;
    }
    // lower triangle, scaled into [-1, 1]
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < n; ++i) mat(i, j) = (i >= j) ? a.coeff(i, j) : 0.0;
    double scale = mat.cwiseAbs().maxCoeff();
    if (scale == 0.0) scale = 1.0;
    for (Index j = 0; j < n; ++j)
      for (Index i = j; i < n; ++i) mat(i, j) /= scale;
    std::vector<double> sub(static_cast<std::size_t>(n - 1));
    if (n == 3)
      tridiag3(mat, diag, sub, vecs);
    else
      tridiag_householder(mat, diag, sub, vecs);
    // computeFromTridiagonal_impl
    Index end = n - 1, start = 0, iter = 0;
    const int max_iter = 30;
    const double zero = std::numeric_limits<double>::min();
    const double prec_inv = 1.0 / std::numeric_limits<double>::epsilon();
    while (end > 0) {
      for (Index i = start; i < end; ++i) {
        if (std::abs(sub[static_cast<std::size_t>(i)]) < zero) {
          sub[static_cast<std::size_t>(i)] = 0.0;
        } else {
          const double scaled = prec_inv * sub[static_cast<std::size_t>(i)];
          if (scaled * scaled <= (std::abs(diag(i)) + std::abs(diag(i + 1)))) sub[static_cast<std::size_t>(i)] = 0.0;
        }
      }
      while (end > 0 && sub[static_cast<std::size_t>(end - 1)] == 0.0) end--;
      if (end <= 0) break;
      iter++;
      if (iter > max_iter * n) break;
      start = end - 1;
      while (start > 0 && sub[static_cast<std::size_t>(start - 1)] != 0.0) start--;
      internal::tridiagonal_qr_step(diag.data(), sub.data(), start, end, vecs ? &mat : nullptr);
    }
    info_ = (iter <= max_iter * n) ? Success : NoConvergence;
    if (info_ == Success) {
      for (Index i = 0; i < n - 1; ++i) {
        Index k = 0;
        diag.segment(i, n - i).minCoeff(&k);
        if (k > 0) {
          std::swap(diag(i), diag(k + i));
          if (vecs) mat.col(i).swap(mat.col(k + i));
        }
      }
    }
    diag *= scale;
    eivalues_ = diag;
    eivec_ = mat;
    return *this;
  }
  const EV& eigenvalues() const { return eivalues_; }
  const MatrixType& eigenvectors() const { return eivec_; }
  ComputationInfo info() const { return info_; }

 private:
  // tridiagonalization_inplace_selector<MatrixType, 3, false>
  static void tridiag3(MatrixXd& mat, VectorXd& diag, std::vector<double>& sub, bool extractQ) {
    const double tol = std::numeric_limits<double>::min();
    diag(0) = mat(0, 0);
    const double v1norm2 = mat(2, 0) * mat(2, 0);
    if (v1norm2 <= tol) {
      diag(1) = mat(1, 1);
      diag(2) = mat(2, 2);
      sub[0] = mat(1, 0);
      sub[1] = mat(2, 1);
      if (extractQ) mat.setIdentity();
    } else {
      const double beta = std::sqrt(mat(1, 0) * mat(1, 0) + v1norm2);
      const double inv_beta = 1.0 / beta;
      const double m01 = mat(1, 0) * inv_beta;
      const double m02 = mat(2, 0) * inv_beta;
      const double q = 2.0 * m01 * mat(2, 1) + m02 * (mat(2, 2) - mat(1, 1));
      diag(1) = mat(1, 1) + m02 * q;
      diag(2) = mat(2, 2) - m02 * q;
      sub[0] = beta;
      sub[1] = mat(2, 1) - m01 * q;
      if (extractQ) {
        mat.setZero();
        mat(0, 0) = 1.0;
        mat(1, 1) = m01;
        mat(1, 2) = m02;
        mat(2, 1) = m02;
        mat(2, 2) = -m01;
      }
    }
  }
  // general Householder tridiagonalization (Tridiagonalization.h), lower
  // triangle stored; Q accumulated explicitly when requested.
  static void tridiag_householder(MatrixXd& a, VectorXd& diag, std::vector<double>& sub, bool extractQ) {
    const Index n = a.rows();
    // full symmetric copy from the lower triangle
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < j; ++i) a(i, j) = a(j, i);
    MatrixXd q = MatrixXd::Identity(n, n);
    for (Index i = 0; i < n - 1; ++i) {
      const Index rem = n - i - 1;
      // makeHouseholderInPlace on a(i+1.., i)
      double tail_sq = 0.0;
      for (Index k = i + 2; k < n; ++k) tail_sq += a(k, i) * a(k, i);
      const double c0 = a(i + 1, i);
      double tau = 0.0, beta = c0;
      std::vector<double> v(static_cast<std::size_t>(rem), 0.0);
      v[0] = 1.0;
      if (tail_sq <= std::numeric_limits<double>::min()) {
        tau = 0.0;
        beta = c0;
      } else {
        beta = std::sqrt(c0 * c0 + tail_sq);
        if (c0 >= 0.0) beta = -beta;
        for (Index k = 1; k < rem; ++k) v[static_cast<std::size_t>(k)] = a(i + 1 + k, i) / (c0 - beta);
        tau = (beta - c0) / beta;
      }
      // A22 <- H A22 H, H = I - tau v v^T
      if (tau != 0.0) {
        std::vector<double> p(static_cast<std::size_t>(rem), 0.0);
        for (Index r = 0; r < rem; ++r) {
          double s = 0.0;
          for (Index c = 0; c < rem; ++c) s += a(i + 1 + r, i + 1 + c) * v[static_cast<std::size_t>(c)];
          p[static_cast<std::size_t>(r)] = tau * s;
        }
        double vp = 0.0;
        for (Index r = 0; r < rem; ++r) vp += v[static_cast<std::size_t>(r)] * p[static_cast<std::size_t>(r)];
        const double alpha = -0.5 * tau * vp;
        for (Index r = 0; r < rem; ++r) p[static_cast<std::size_t>(r)] += alpha * v[static_cast<std::size_t>(r)];
        for (Index c = 0; c < rem; ++c)
          for (Index r = 0; r < rem; ++r)
            a(i + 1 + r, i + 1 + c) -= v[static_cast<std::size_t>(r)] * p[static_cast<std::size_t>(c)] +
                                       p[static_cast<std::size_t>(r)] * v[static_cast<std::size_t>(c)];
        if (extractQ) {
          // q <- q H (columns i+1..)
          for (Index r = 0; r < n; ++r) {
            double s = 0.0;
            for (Index c = 0; c < rem; ++c) s += q(r, i + 1 + c) * v[static_cast<std::size_t>(c)];
            s *= tau;
            for (Index c = 0; c < rem; ++c) q(r, i + 1 + c) -= s * v[static_cast<std::size_t>(c)];
          }
        }
      }
      sub[static_cast<std::size_t>(i)] = beta;
      diag(i) = a(i, i);
    }
    diag(n - 1) = a(n - 1, n - 1);
    a = q;
  }

  EV eivalues_;
  MatrixType eivec_;
  ComputationInfo info_ = Success;
};

// ---------------------------------------------------------------------------
// JacobiSVD (two-sided Jacobi on square matrices)
template <class MatrixType>
class JacobiSVD {
 public:
  template <DenseExpr E>
  JacobiSVD(const E& a, int /*options*/ = 0) {
    const Index n = a.rows();
    MatrixXd w(a);
    MatrixXd u = MatrixXd::Identity(n, n), v = MatrixXd::Identity(n, n);
    for (int sweep = 0; sweep < 60; ++sweep) {
      bool done = true;
      for (Index p = 1; p < n; ++p)
        for (Index q = 0; q < p; ++q) {
          const double thr = std::max(2.0 * std::numeric_limits<double>::denorm_min(),
                                      2.0 * std::numeric_limits<double>::epsilon() *
                                          std::max(std::abs(w(p, p)), std::abs(w(q, q))));
          if (std::abs(w(p, q)) > thr || std::abs(w(q, p)) > thr) {
            done = false;
            // symmetrise the 2x2 block with a left rotation, then diagonalise
            const double t = w(p, p) + w(q, q), d = w(q, p) - w(p, q);
            double c1 = 1.0, s1 = 0.0;
            if (std::abs(d) > std::numeric_limits<double>::min()) {
              const double u1 = t / d, tmp = std::sqrt(1.0 + u1 * u1);
              s1 = 1.0 / tmp;
              c1 = u1 * s1;
            }
            // rot1 applied on the left to rows (p, q)
            for (Index c = 0; c < n; ++c) {
              const double x = w(p, c), y = w(q, c);
              w(p, c) = c1 * x + s1 * y;
              w(q, c) = -s1 * x + c1 * y;
            }
            for (Index r = 0; r < n; ++r) {
              const double x = u(r, p), y = u(r, q);
              u(r, p) = c1 * x + s1 * y;
              u(r, q) = -s1 * x + c1 * y;
            }
            // symmetric 2x2 Jacobi on (p, q)
            const double app = w(p, p), aqq = w(q, q), apq = w(p, q);
            if (apq != 0.0) {
              const double tau = (aqq - app) / (2.0 * apq);
              const double tt = (tau >= 0 ? 1.0 : -1.0) / (std::abs(tau) + std::sqrt(1.0 + tau * tau));
              const double c = 1.0 / std::sqrt(1.0 + tt * tt), s = tt * c;
              for (Index cc = 0; cc < n; ++cc) {
                const double x = w(p, cc), y = w(q, cc);
                w(p, cc) = c * x - s * y;
                w(q, cc) = s * x + c * y;
              }
              for (Index r = 0; r < n; ++r) {
                const double x = w(r, p), y = w(r, q);
                w(r, p) = c * x - s * y;
                w(r, q) = s * x + c * y;
              }
              for (Index r = 0; r < n; ++r) {
                const double x = u(r, p), y = u(r, q);
                u(r, p) = c * x - s * y;
                u(r, q) = s * x + c * y;
              }
              for (Index r = 0; r < n; ++r) {
                const double x = v(r, p), y = v(r, q);
                v(r, p) = c * x - s * y;
                v(r, q) = s * x + c * y;
              }
            }
          }
        }
      if (done) break;
    }
    // singular values non-negative, sorted descending
    sv_.resize(n);
    for (Index i = 0; i < n; ++i) {
      sv_(i) = std::abs(w(i, i));
      if (w(i, i) < 0.0) u.col(i) *= -1.0;
    }
    for (Index i = 0; i < n; ++i) {
      Index best = i;
      for (Index k = i + 1; k < n; ++k)
        if (sv_(k) > sv_(best)) best = k;
      if (best != i) {
        std::swap(sv_(i), sv_(best));
        u.col(i).swap(u.col(best));
        v.col(i).swap(v.col(best));
      }
    }
    u_ = u;
    v_ = v;
  }
  const MatrixType& matrixU() const { return u_; }
  const MatrixType& matrixV() const { return v_; }
  const VectorXd& singularValues() const { return sv_; }

 private:
  MatrixType u_, v_;
  VectorXd sv_;
};

// ---------------------------------------------------------------------------
// Geometry: AngleAxis, Quaternion, Transform (Isometry)
template <class S>
class AngleAxis {
 public:
  AngleAxis() = default;
  template <DenseExpr E>
  AngleAxis(double angle, const E& axis) : angle_(angle), axis_(axis) {}
  double angle() const { return angle_; }
  const Vector3d& axis() const { return axis_; }
  Matrix3d toRotationMatrix() const {
    Matrix3d res;
    const Vector3d sin_axis = std::sin(angle_) * axis_;
    const double c = std::cos(angle_);
    const Vector3d cos1_axis = (1.0 - c) * axis_;
    double tmp = cos1_axis.x() * axis_.y();
    res(0, 1) = tmp - sin_axis.z();
    res(1, 0) = tmp + sin_axis.z();
    tmp = cos1_axis.x() * axis_.z();
    res(0, 2) = tmp + sin_axis.y();
    res(2, 0) = tmp - sin_axis.y();
    tmp = cos1_axis.y() * axis_.z();
    res(1, 2) = tmp - sin_axis.x();
    res(2, 1) = tmp + sin_axis.x();
    for (int i = 0; i < 3; ++i) res(i, i) = cos1_axis(i) * axis_(i) + c;
    return res;
  }
  Matrix3d matrix() const { return toRotationMatrix(); }

 private:
  double angle_ = 0.0;
  Vector3d axis_ = Vector3d::UnitX();
};
using AngleAxisd = AngleAxis<double>;

template <class S>
class Quaternion {
 public:
  Quaternion() = default;
  Quaternion(double w, double x, double y, double z) : w_(w), v_(x, y, z) {}
  Quaternion(const AngleAxis<S>& aa) {
    const double ha = 0.5 * aa.angle();
    w_ = std::cos(ha);
    v_ = std::sin(ha) * aa.axis();
  }
  // from a rotation matrix (Eigen's quaternionbase_assign_impl<Matrix3>)
  template <DenseExpr E>
  explicit Quaternion(const E& m) {
    const double t = m.trace();
    if (t > 0.0) {
      double tt = std::sqrt(t + 1.0);
      w_ = 0.5 * tt;
      tt = 0.5 / tt;
      v_(0) = (m.coeff(2, 1) - m.coeff(1, 2)) * tt;
      v_(1) = (m.coeff(0, 2) - m.coeff(2, 0)) * tt;
      v_(2) = (m.coeff(1, 0) - m.coeff(0, 1)) * tt;
    } else {
      Index i = 0;
      if (m.coeff(1, 1) > m.coeff(0, 0)) i = 1;
      if (m.coeff(2, 2) > m.coeff(i, i)) i = 2;
      const Index j = (i + 1) % 3, k = (j + 1) % 3;
      double tt = std::sqrt(m.coeff(i, i) - m.coeff(j, j) - m.coeff(k, k) + 1.0);
      v_(i) = 0.5 * tt;
      tt = 0.5 / tt;
      w_ = (m.coeff(k, j) - m.coeff(j, k)) * tt;
      v_(j) = (m.coeff(j, i) + m.coeff(i, j)) * tt;
      v_(k) = (m.coeff(k, i) + m.coeff(i, k)) * tt;
    }
  }
  double w() const { return w_; }
  double x() const { return v_(0); }
  double y() const { return v_(1); }
  double z() const { return v_(2); }
  double& w() { return w_; }
  double& x() { return v_(0); }
  double& y() { return v_(1); }
  double& z() { return v_(2); }
  const Vector3d& vec() const { return v_; }
  Quaternion normalized() const {
    const double n = std::sqrt(w_ * w_ + v_.squaredNorm());
    return Quaternion(w_ / n, v_(0) / n, v_(1) / n, v_(2) / n);
  }
  void normalize() { *this = normalized(); }
  Quaternion conjugate() const { return Quaternion(w_, -v_(0), -v_(1), -v_(2)); }
  Quaternion inverse() const { return conjugate(); }
  Matrix3d toRotationMatrix() const {
    Matrix3d res;
    const double tx = 2.0 * x(), ty = 2.0 * y(), tz = 2.0 * z();
    const double twx = tx * w(), twy = ty * w(), twz = tz * w();
    const double txx = tx * x(), txy = ty * x(), txz = tz * x();
    const double tyy = ty * y(), tyz = tz * y(), tzz = tz * z();
    res(0, 0) = 1.0 - (tyy + tzz);
    res(0, 1) = txy - twz;
    res(0, 2) = txz + twy;
    res(1, 0) = txy + twz;
    res(1, 1) = 1.0 - (txx + tzz);
    res(1, 2) = tyz - twx;
    res(2, 0) = txz - twy;
    res(2, 1) = tyz + twx;
    res(2, 2) = 1.0 - (txx + tyy);
    return res;
  }
  Matrix3d matrix() const { return toRotationMatrix(); }
  friend Quaternion operator*(const Quaternion& a, const Quaternion& b) {
    return Quaternion(a.w() * b.w() - a.x() * b.x() - a.y() * b.y() - a.z() * b.z(),
                      a.w() * b.x() + a.x() * b.w() + a.y() * b.z() - a.z() * b.y(),
                      a.w() * b.y() + a.y() * b.w() + a.z() * b.x() - a.x() * b.z(),
                      a.w() * b.z() + a.z() * b.w() + a.x() * b.y() - a.y() * b.x());
  }
  template <DenseExpr E>
  Vector3d operator*(const E& v) const {
    return toRotationMatrix() * v;
  }

 private:
  double w_ = 1.0;
  Vector3d v_ = Vector3d::Zero();
};
using Quaterniond = Quaternion<double>;

template <class S>
Quaternion<S> operator*(const AngleAxis<S>& a, const AngleAxis<S>& b) {
  return Quaternion<S>(a) * Quaternion<S>(b);
}

template <class S, int Dim, int Mode>
class Transform {
 public:
  static Transform Identity() { return Transform(); }
  View<3, 1, false> translation() { return View<3, 1, false>(t_.data(), 3, 1, 1, 3); }
  const Vector3d& translation() const { return t_; }
  Matrix3d& linear() { return l_; }
  const Matrix3d& linear() const { return l_; }
  Matrix3d rotation() const { return l_; }
  template <DenseExpr E>
  Transform& translate(const E& v) {
    t_ += l_ * v;
    return *this;
  }
  Transform& rotate(const AngleAxis<S>& aa) {
    l_ = l_ * aa.toRotationMatrix();
    return *this;
  }
  template <DenseExpr E>
  Transform& rotate(const E& r) {
    l_ = l_ * r;
    return *this;
  }
  template <DenseExpr E>
  Vector3d operator*(const E& p) const {
    return l_ * p + t_;
  }
  Transform operator*(const Transform& o) const {
    Transform r;
    r.l_ = l_ * o.l_;
    r.t_ = l_ * o.t_ + t_;
    return r;
  }
  Transform inverse() const {
    Transform r;
    r.l_ = l_.transpose();
    r.t_ = -(r.l_ * t_);
    return r;
  }

 private:
  Matrix3d l_ = Matrix3d::Identity();
  Vector3d t_ = Vector3d::Zero();
};
using Isometry3d = Transform<double, 3, Isometry>;
using Affine3d = Transform<double, 3, Affine>;

}  // namespace Eigen
