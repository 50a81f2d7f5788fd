// Eigen-subset — TEST INFRASTRUCTURE ONLY. Definitions of the Ops members and
// the free operators declared in Eigen/Core (see its header for the
// evaluation-order contract).
#pragma once

namespace Eigen {

namespace internal {

template <class T> struct is_ops_d : is_ops<std::remove_cv_t<std::remove_reference_t<T>>> {};
template <class A, class B = void> using if_ops = std::enable_if_t<is_ops_d<A>::value, B>;
template <class A, class B> using if_ops2 = std::enable_if_t<is_ops_d<A>::value && is_ops_d<B>::value, int>;
template <class A, class T> using if_ops_scalar =
    std::enable_if_t<is_ops_d<A>::value && std::is_arithmetic_v<std::remove_cv_t<std::remove_reference_t<T>>>, int>;

template <class D> auto to_dyn(const D& d) { return dyn_t<D>(d); }

template <class T, class D, class F> auto cw(const D& d, F f) { return map1<T>(d, f); }

// Matrix inverse: explicit 2x2 formula (Eigen's compute_inverse<2x2>),
// partial-pivot LU otherwise.
template <class M> M inverse_of(const M& m) {
  const Index n = m.rows();
  if (n != m.cols()) throw std::logic_error("Eigen-subset: inverse of a non-square matrix");
  M r(m);
  if (n == 2) {
    const double det = m.coeff(0, 0) * m.coeff(1, 1) - m.coeff(1, 0) * m.coeff(0, 1);
    const double invdet = 1.0 / det;
    r.coeffRef(0, 0) = m.coeff(1, 1) * invdet;
    r.coeffRef(1, 0) = -m.coeff(1, 0) * invdet;
    r.coeffRef(0, 1) = -m.coeff(0, 1) * invdet;
    r.coeffRef(1, 1) = m.coeff(0, 0) * invdet;
    return r;
  }
  std::vector<double> a(std::size_t(n * n)), inv(std::size_t(n * n), 0.0);
  for (Index i = 0; i < n; ++i)
    for (Index j = 0; j < n; ++j) a[std::size_t(i * n + j)] = m.coeff(i, j);
  std::vector<Index> perm(static_cast<std::size_t>(n));
  std::iota(perm.begin(), perm.end(), Index(0));
  for (Index k = 0; k < n; ++k) {
    Index piv = k;
    for (Index i = k + 1; i < n; ++i)
      if (std::abs(a[std::size_t(i * n + k)]) > std::abs(a[std::size_t(piv * n + k)])) piv = i;
    if (piv != k) {
      for (Index j = 0; j < n; ++j) std::swap(a[std::size_t(k * n + j)], a[std::size_t(piv * n + j)]);
      std::swap(perm[std::size_t(k)], perm[std::size_t(piv)]);
    }
    const double d = a[std::size_t(k * n + k)];
    for (Index i = k + 1; i < n; ++i) {
      a[std::size_t(i * n + k)] /= d;
      for (Index j = k + 1; j < n; ++j) a[std::size_t(i * n + j)] -= a[std::size_t(i * n + k)] * a[std::size_t(k * n + j)];
    }
  }
  for (Index c = 0; c < n; ++c) {
    std::vector<double> x(static_cast<std::size_t>(n));
    for (Index i = 0; i < n; ++i) x[std::size_t(i)] = perm[std::size_t(i)] == c ? 1.0 : 0.0;
    for (Index i = 0; i < n; ++i)
      for (Index j = 0; j < i; ++j) x[std::size_t(i)] -= a[std::size_t(i * n + j)] * x[std::size_t(j)];
    for (Index i = n - 1; i >= 0; --i) {
      for (Index j = i + 1; j < n; ++j) x[std::size_t(i)] -= a[std::size_t(i * n + j)] * x[std::size_t(j)];
      x[std::size_t(i)] /= a[std::size_t(i * n + i)];
    }
    for (Index i = 0; i < n; ++i) r.coeffRef(i, c) = x[std::size_t(i)];
  }
  return r;
}

}  // namespace internal

template <class D> auto Ops<D>::eval() const { return internal::to_dyn(derived()); }
template <class D> auto Ops<D>::array() const { return internal::dyn_kind<D, true>(derived()); }
template <class D> auto Ops<D>::matrix() const { return internal::dyn_kind<D, false>(derived()); }
template <class D> auto Ops<D>::transpose() const {
  using S = internal::scalar_t<D>;
  const D& d = derived();
  Dense<S, Dynamic, Dynamic, D::IsRowMajor ? 0 : 1, D::IsArray> r(d.cols(), d.rows());
  for (Index i = 0; i < d.rows(); ++i)
    for (Index j = 0; j < d.cols(); ++j) r.coeffRef(j, i) = d.coeff(i, j);
  return r;
}
template <class D> template <class T> auto Ops<D>::cast() const {
  return internal::map1<T>(derived(), [](auto v) { return T(v); });
}
template <class D> auto Ops<D>::rowwise() const { return VectorwiseOp<internal::dyn_t<D>>(eval(), false); }
template <class D> auto Ops<D>::colwise() const { return VectorwiseOp<internal::dyn_t<D>>(eval(), true); }

template <class D> auto Ops<D>::cwiseAbs() const {
  using S = internal::scalar_t<D>;
  return internal::map1<S>(derived(), [](S v) { return std::abs(v); });
}
template <class D> auto Ops<D>::cwiseAbs2() const {
  using S = internal::scalar_t<D>;
  return internal::map1<S>(derived(), [](S v) { return v * v; });
}
template <class D> auto Ops<D>::cwiseSqrt() const {
  using S = internal::scalar_t<D>;
  return internal::map1<S>(derived(), [](S v) { return std::sqrt(v); });
}
template <class D> auto Ops<D>::cwiseInverse() const {
  using S = internal::scalar_t<D>;
  return internal::map1<S>(derived(), [](S v) { return S(1) / v; });
}
template <class D> auto Ops<D>::exp() const {
  using S = internal::scalar_t<D>;
  return internal::map1<S>(derived(), [](S v) { return std::exp(v); });
}
template <class D> auto Ops<D>::log() const {
  using S = internal::scalar_t<D>;
  return internal::map1<S>(derived(), [](S v) { return std::log(v); });
}
template <class D> auto Ops<D>::inverse() const {
  if constexpr (D::IsArray) {
    return cwiseInverse();
  } else {
    return internal::inverse_of(eval());
  }
}
template <class D> template <class O> auto Ops<D>::cwiseProduct(const O& o) const {
  using S = internal::scalar_t<D>;
  return internal::map2<S>(derived(), o, [](S a, S b) { return a * b; });
}
template <class D> template <class O> auto Ops<D>::cwiseQuotient(const O& o) const {
  using S = internal::scalar_t<D>;
  return internal::map2<S>(derived(), o, [](S a, S b) { return a / b; });
}
template <class D> template <class O> auto Ops<D>::cwiseMax(const O& o) const {
  using S = internal::scalar_t<D>;
  if constexpr (std::is_arithmetic_v<O>) {
    const S b = S(o);
    return internal::map1<S>(derived(), [b](S a) { return std::max(a, b); });
  } else {
    return internal::map2<S>(derived(), o, [](S a, S b) { return std::max(a, b); });
  }
}
template <class D> template <class O> auto Ops<D>::cwiseMin(const O& o) const {
  using S = internal::scalar_t<D>;
  if constexpr (std::is_arithmetic_v<O>) {
    const S b = S(o);
    return internal::map1<S>(derived(), [b](S a) { return std::min(a, b); });
  } else {
    return internal::map2<S>(derived(), o, [](S a, S b) { return std::min(a, b); });
  }
}
template <class D> auto Ops<D>::isFinite() const {
  using S = internal::scalar_t<D>;
  return internal::map1<bool>(derived(), [](S v) { return bool(std::isfinite(v)); });
}
template <class D> auto Ops<D>::isNaN() const {
  using S = internal::scalar_t<D>;
  return internal::map1<bool>(derived(), [](S v) { return bool(std::isnan(v)); });
}
template <class D> auto Ops<D>::operator-() const {
  using S = internal::scalar_t<D>;
  return internal::map1<S>(derived(), [](S v) { return -v; });
}

// The object's compile-time size when it is a fixed-size plain object.
template <class D> constexpr int fixed_size_of_v() {
  if constexpr (D::SizeAtCompileTime != Dynamic) return D::SizeAtCompileTime;
  else return 0;
}

template <class D> auto Ops<D>::sum() const {
  return internal::redux_sum(derived(), false, fixed_size_of_v<D>());
}
template <class D> auto Ops<D>::prod() const {
  auto r = lin(0);
  for (Index k = 1; k < size(); ++k) r = r * lin(k);
  return r;
}
template <class D> auto Ops<D>::mean() const {
  using S = internal::scalar_t<D>;
  return sum() / S(size());
}
template <class D> auto Ops<D>::squaredNorm() const {
  // cwiseAbs2() of the object is an expression: aligned start 0; its
  // traversal follows the object's (contiguous or strided) layout.
  using S = internal::scalar_t<D>;
  const D& d = derived();
  const Index n = d.rows() * d.cols();
  if (n == 0) return S(0);
  if constexpr (fixed_size_of_v<D>() > 0) {
    // cost = size * (read 1 + mul 1) + (size - 1) adds, unrolled when <= 220
    if (fixed_size_of_v<D>() * 3 - 1 <= 220) {
      std::vector<double> v(static_cast<std::size_t>(n));
      for (Index k = 0; k < n; ++k) v[std::size_t(k)] = double(d.lin(k)) * double(d.lin(k));
      return S(internal::unrolled_sum(v.data(), n));
    }
  }
  if (d.contiguous()) {
    std::vector<double> v(static_cast<std::size_t>(n));
    Index k = 0;
    if (d.root_row_major())
      for (Index i = 0; i < d.rows(); ++i)
        for (Index j = 0; j < d.cols(); ++j) v[std::size_t(k++)] = d.coeff(i, j) * d.coeff(i, j);
    else
      for (Index j = 0; j < d.cols(); ++j)
        for (Index i = 0; i < d.rows(); ++i) v[std::size_t(k++)] = d.coeff(i, j) * d.coeff(i, j);
    return S(internal::packet_sum(v.data(), n, 0));
  }
  S r = d.lin(0) * d.lin(0);
  for (Index k = 1; k < n; ++k) r = r + d.lin(k) * d.lin(k);
  return r;
}
template <class D> auto Ops<D>::norm() const { return std::sqrt(squaredNorm()); }
template <class D> template <class O> auto Ops<D>::dot(const O& o) const {
  // Eigen: (a.conjugate().cwiseProduct(b)).sum() — an expression over both.
  auto p = cwiseProduct(o);
  return internal::redux_sum(p, true, 0);
}
template <class D> auto Ops<D>::maxCoeff() const {
  auto r = lin(0);
  for (Index k = 1; k < size(); ++k)
    if (lin(k) > r) r = lin(k);
  return r;
}
template <class D> auto Ops<D>::minCoeff() const {
  auto r = lin(0);
  for (Index k = 1; k < size(); ++k)
    if (lin(k) < r) r = lin(k);
  return r;
}
template <class D> template <class I> auto Ops<D>::maxCoeff(I* idx) const {
  Index best = 0;
  for (Index k = 1; k < size(); ++k)
    if (lin(k) > lin(best)) best = k;
  *idx = I(best);
  return lin(best);
}
template <class D> template <class I> auto Ops<D>::minCoeff(I* idx) const {
  Index best = 0;
  for (Index k = 1; k < size(); ++k)
    if (lin(k) < lin(best)) best = k;
  *idx = I(best);
  return lin(best);
}
template <class D> template <class I> auto Ops<D>::maxCoeff(I* ri, I* ci) const {
  const D& d = derived();
  Index bi = 0, bj = 0;
  for (Index j = 0; j < d.cols(); ++j)
    for (Index i = 0; i < d.rows(); ++i)
      if (d.coeff(i, j) > d.coeff(bi, bj)) {
        bi = i;
        bj = j;
      }
  *ri = I(bi);
  *ci = I(bj);
  return d.coeff(bi, bj);
}
template <class D> template <class I> auto Ops<D>::minCoeff(I* ri, I* ci) const {
  const D& d = derived();
  Index bi = 0, bj = 0;
  for (Index j = 0; j < d.cols(); ++j)
    for (Index i = 0; i < d.rows(); ++i)
      if (d.coeff(i, j) < d.coeff(bi, bj)) {
        bi = i;
        bj = j;
      }
  *ri = I(bi);
  *ci = I(bj);
  return d.coeff(bi, bj);
}
template <class D> bool Ops<D>::all() const {
  for (Index k = 0; k < size(); ++k)
    if (!bool(lin(k))) return false;
  return true;
}
template <class D> bool Ops<D>::any() const {
  for (Index k = 0; k < size(); ++k)
    if (bool(lin(k))) return true;
  return false;
}
template <class D> Index Ops<D>::count() const {
  Index c = 0;
  for (Index k = 0; k < size(); ++k) c += bool(lin(k)) ? 1 : 0;
  return c;
}
template <class D> bool Ops<D>::allFinite() const { return isFinite().all(); }
template <class D> bool Ops<D>::hasNaN() const { return isNaN().any(); }

// ---------------------------------------------------------------- products
namespace internal {

template <class DA, class DB>
auto product(const DA& a, const DB& b) {
  using S = scalar_t<DA>;
  if (a.cols() != b.rows()) throw std::logic_error("Eigen-subset: product size mismatch");
  using R = Dense<S, DA::RowsAtCompileTime, DB::ColsAtCompileTime, 0, false>;
  auto r = make_result<R>(a.rows(), b.cols());
  const Index K = a.cols();
  const bool lazy = (DA::SizeAtCompileTime != Dynamic && DB::SizeAtCompileTime != Dynamic) ||
                    (b.rows() + a.rows() + b.cols() < 20 && b.rows() > 0);
  for (Index i = 0; i < a.rows(); ++i)
    for (Index j = 0; j < b.cols(); ++j) {
      S acc;
      if (K == 0) {
        acc = S(0);
      } else if (lazy) {  // coefficient-based: first product, then k ascending
        acc = a.coeff(i, 0) * b.coeff(0, j);
        for (Index k = 1; k < K; ++k) acc = acc + a.coeff(i, k) * b.coeff(k, j);
      } else {  // GEMM/GEMV: zero accumulator, k ascending, added to a zeroed destination
        acc = S(0);
        for (Index k = 0; k < K; ++k) acc = acc + a.coeff(i, k) * b.coeff(k, j);
        acc = S(0) + acc;
      }
      r.coeffRef(i, j) = acc;
    }
  return r;
}

}  // namespace internal

// ---------------------------------------------------------------- operators
#define EIGEN_SUBSET_BINOP(OP)                                                                         \
  template <class A, class B, internal::if_ops2<A, B> = 0>                                           \
  auto operator OP(const A& a, const B& b) {                                                         \
    using S = internal::scalar_t<A>;                                                                 \
    return internal::map2<S>(a, b, [](S x, S y) { return x OP y; });                                 \
  }                                                                                                  \
  template <class A, class T, internal::if_ops_scalar<A, T> = 0>                                     \
  auto operator OP(const A& a, T t) {                                                                \
    using S = internal::scalar_t<A>;                                                                 \
    const S y = S(t);                                                                                \
    return internal::map1<S>(a, [y](S x) { return x OP y; });                                        \
  }                                                                                                  \
  template <class A, class T, internal::if_ops_scalar<A, T> = 0>                                     \
  auto operator OP(T t, const A& a) {                                                                \
    using S = internal::scalar_t<A>;                                                                 \
    const S y = S(t);                                                                                \
    return internal::map1<S>(a, [y](S x) { return y OP x; });                                        \
  }

EIGEN_SUBSET_BINOP(+)
EIGEN_SUBSET_BINOP(-)
EIGEN_SUBSET_BINOP(/)
#undef EIGEN_SUBSET_BINOP

template <class A, class B, internal::if_ops2<A, B> = 0>
auto operator*(const A& a, const B& b) {
  using S = internal::scalar_t<A>;
  if constexpr (A::IsArray) {
    return internal::map2<S>(a, b, [](S x, S y) { return x * y; });
  } else {
    return internal::product(a, b);
  }
}
template <class A, class T, internal::if_ops_scalar<A, T> = 0>
auto operator*(const A& a, T t) {
  using S = internal::scalar_t<A>;
  const S y = S(t);
  return internal::map1<S>(a, [y](S x) { return x * y; });
}
template <class A, class T, internal::if_ops_scalar<A, T> = 0>
auto operator*(T t, const A& a) {
  using S = internal::scalar_t<A>;
  const S y = S(t);
  return internal::map1<S>(a, [y](S x) { return y * x; });
}

#define EIGEN_SUBSET_CMP(OP)                                                                         \
  template <class A, class B, internal::if_ops2<A, B> = 0>                                           \
  auto operator OP(const A& a, const B& b) {                                                         \
    using S = internal::scalar_t<A>;                                                                 \
    return internal::map2<bool>(a, b, [](S x, S y) { return x OP y; });                              \
  }                                                                                                  \
  template <class A, class T, internal::if_ops_scalar<A, T> = 0>                                     \
  auto operator OP(const A& a, T t) {                                                                \
    using S = internal::scalar_t<A>;                                                                 \
    const S y = S(t);                                                                                \
    return internal::map1<bool>(a, [y](S x) { return x OP y; });                                     \
  }

EIGEN_SUBSET_CMP(<)
EIGEN_SUBSET_CMP(<=)
EIGEN_SUBSET_CMP(>)
EIGEN_SUBSET_CMP(>=)
#undef EIGEN_SUBSET_CMP

// == / != : coefficient-wise for arrays, a single bool for matrices.
template <class A, class B, internal::if_ops2<A, B> = 0>
auto operator==(const A& a, const B& b) {
  using S = internal::scalar_t<A>;
  if constexpr (A::IsArray) {
    return internal::map2<bool>(a, b, [](S x, S y) { return x == y; });
  } else {
    if (a.rows() != b.rows() || a.cols() != b.cols()) return false;
    return internal::map2<bool>(a, b, [](S x, S y) { return x == y; }).all();
  }
}
template <class A, class B, internal::if_ops2<A, B> = 0>
auto operator!=(const A& a, const B& b) {
  using S = internal::scalar_t<A>;
  if constexpr (A::IsArray) {
    return internal::map2<bool>(a, b, [](S x, S y) { return x != y; });
  } else {
    return !(a == b);
  }
}
template <class A, class T, internal::if_ops_scalar<A, T> = 0>
auto operator==(const A& a, T t) {
  using S = internal::scalar_t<A>;
  const S y = S(t);
  return internal::map1<bool>(a, [y](S x) { return x == y; });
}
template <class A, class T, internal::if_ops_scalar<A, T> = 0>
auto operator!=(const A& a, T t) {
  using S = internal::scalar_t<A>;
  const S y = S(t);
  return internal::map1<bool>(a, [y](S x) { return x != y; });
}

template <class A, class B, internal::if_ops2<A, B> = 0>
auto operator&&(const A& a, const B& b) {
  return internal::map2<bool>(a, b, [](bool x, bool y) { return x && y; });
}
template <class A, class B, internal::if_ops2<A, B> = 0>
auto operator||(const A& a, const B& b) {
  return internal::map2<bool>(a, b, [](bool x, bool y) { return x || y; });
}

// ---------------------------------------------------------------- compound assignment
template <class S, int R, int C, int RM, bool A>
template <class O>
Dense<S, R, C, RM, A>& Dense<S, R, C, RM, A>::operator+=(const O& o) {
  if constexpr (std::is_arithmetic_v<O>) {
    for (auto& v : d_) v = v + S(o);
  } else {
    assign(internal::map2<S>(*this, o, [](S x, S y) { return x + y; }));
  }
  return *this;
}
template <class S, int R, int C, int RM, bool A>
template <class O>
Dense<S, R, C, RM, A>& Dense<S, R, C, RM, A>::operator-=(const O& o) {
  if constexpr (std::is_arithmetic_v<O>) {
    for (auto& v : d_) v = v - S(o);
  } else {
    assign(internal::map2<S>(*this, o, [](S x, S y) { return x - y; }));
  }
  return *this;
}
template <class P>
template <class O>
Block<P>& Block<P>::operator+=(const O& o) {
  return assign(internal::map2<S>(*this, o, [](S x, S y) { return x + y; }));
}
template <class P>
template <class O>
Block<P>& Block<P>::operator-=(const O& o) {
  return assign(internal::map2<S>(*this, o, [](S x, S y) { return x - y; }));
}

template <class D>
std::ostream& operator<<(std::ostream& os, const Ops<D>& m) {
  const D& d = m.derived();
  for (Index i = 0; i < d.rows(); ++i) {
    for (Index j = 0; j < d.cols(); ++j) os << (j ? " " : "") << d.coeff(i, j);
    if (i + 1 < d.rows()) os << "\n";
  }
  return os;
}

// ---------------------------------------------------------------- comma initializer
template <class M>
class CommaInitializer {  // m << a, b, c ...: row-major fill
 public:
  CommaInitializer(M& m, typename M::Scalar first) : m_(m) { put(first); }
  CommaInitializer& operator,(typename M::Scalar v) {
    put(v);
    return *this;
  }

 private:
  void put(typename M::Scalar v) {
    m_.coeffRef(k_ / m_.cols(), k_ % m_.cols()) = v;
    ++k_;
  }
  M& m_;
  Index k_ = 0;
};
template <class S, int R, int C, int RM, bool A, class T, std::enable_if_t<std::is_arithmetic_v<T>, int> = 0>
CommaInitializer<Dense<S, R, C, RM, A>> operator<<(Dense<S, R, C, RM, A>& m, T v) {
  return CommaInitializer<Dense<S, R, C, RM, A>>(m, S(v));
}

// ---------------------------------------------------------------- typedefs
template <class S, int R, int C, int Opt = ((R == 1 && C != 1) ? RowMajor : ColMajor), int MR = R, int MC = C>
using Matrix = Dense<S, R, C, (Opt & RowMajor) ? 1 : 0, false>;
template <class S, int R, int C, int Opt = ((R == 1 && C != 1) ? RowMajor : ColMajor), int MR = R, int MC = C>
using Array = Dense<S, R, C, (Opt & RowMajor) ? 1 : 0, true>;

using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using MatrixXi = Matrix<int, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;
using VectorXi = Matrix<int, Dynamic, 1>;
using RowVectorXd = Matrix<double, 1, Dynamic>;
using Matrix2d = Matrix<double, 2, 2>;
using Matrix3d = Matrix<double, 3, 3>;
using Matrix4d = Matrix<double, 4, 4>;
using Vector2d = Matrix<double, 2, 1>;
using Vector3d = Matrix<double, 3, 1>;
using Vector4d = Matrix<double, 4, 1>;
using ArrayXd = Array<double, Dynamic, 1>;
using ArrayXXd = Array<double, Dynamic, Dynamic>;
using ArrayXi = Array<int, Dynamic, 1>;

// Ref<const T>: a by-value evaluation of any compatible expression.
template <class T>
class Ref : public std::remove_const_t<T> {
 public:
  using Base = std::remove_const_t<T>;
  template <class O, std::enable_if_t<internal::is_ops_d<O>::value, int> = 0>
  Ref(const O& o) : Base(o) {}
};
namespace internal {
template <class T> struct is_ops<Ref<T>> : std::true_type {};
}  // namespace internal

}  // namespace Eigen
