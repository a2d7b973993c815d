// linalg.hpp -- fixed-size dense matrices for the shellular drop-in API.
//
// The reference types Vec3/Vec3i/Mat3/Mat6/Mat24 are Eigen typedefs
// (common.hpp:17-21, fem.hpp:32).  Eigen is not a dependency of the B200
// build, so this header provides the subset of Eigen's dense API that code
// written against the reference uses on these types: element access,
// Zero/Identity/Constant, + - * (matrix and scalar), transpose, cwiseAbs,
// min/maxCoeff, norm, dot, cross, cast, segment/block views by value.
// Storage is column-major like Eigen.
#pragma once

#include <algorithm>
#include <cmath>
#include <initializer_list>
#include <type_traits>

namespace shellular {

template <class T, int R, int C>
class Matrix {
 public:
  using Scalar = T;
  static constexpr int RowsAtCompileTime = R;
  static constexpr int ColsAtCompileTime = C;

  Matrix() { setZero(); }
  template <class A, class B, class D,
            class = std::enable_if_t<R * C == 3 && std::is_arithmetic_v<A> &&
                                     std::is_arithmetic_v<B> && std::is_arithmetic_v<D>>>
  Matrix(A a, B b, D d) {
    v_[0] = static_cast<T>(a);
    v_[1] = static_cast<T>(b);
    v_[2] = static_cast<T>(d);
  }

  static Matrix Zero() { return Matrix(); }
  static Matrix Constant(T c) {
    Matrix m;
    m.setConstant(c);
    return m;
  }
  static Matrix Identity() {
    Matrix m;
    for (int i = 0; i < std::min(R, C); ++i) m(i, i) = T(1);
    return m;
  }

  static constexpr int rows() { return R; }
  static constexpr int cols() { return C; }
  static constexpr int size() { return R * C; }

  T& operator()(int i, int j) { return v_[j * R + i]; }
  const T& operator()(int i, int j) const { return v_[j * R + i]; }
  T& operator()(int i) { return v_[i]; }
  const T& operator()(int i) const { return v_[i]; }
  T& operator[](int i) { return v_[i]; }
  const T& operator[](int i) const { return v_[i]; }
  T* data() { return v_; }
  const T* data() const { return v_; }

  Matrix& setZero() { return setConstant(T(0)); }
  Matrix& setConstant(T c) {
    std::fill(v_, v_ + R * C, c);
    return *this;
  }

  Matrix operator+(const Matrix& o) const { return zip(o, [](T a, T b) { return a + b; }); }
  Matrix operator-(const Matrix& o) const { return zip(o, [](T a, T b) { return a - b; }); }
  Matrix operator-() const { return map([](T a) { return -a; }); }
  Matrix& operator+=(const Matrix& o) { return *this = *this + o; }
  Matrix& operator-=(const Matrix& o) { return *this = *this - o; }
  Matrix operator*(T s) const { return map([s](T a) { return a * s; }); }
  Matrix operator/(T s) const { return map([s](T a) { return a / s; }); }
  Matrix& operator*=(T s) { return *this = *this * s; }
  Matrix& operator/=(T s) { return *this = *this / s; }
  friend Matrix operator*(T s, const Matrix& m) { return m * s; }

  template <int C2>
  Matrix<T, R, C2> operator*(const Matrix<T, C, C2>& o) const {
    Matrix<T, R, C2> out;
    for (int j = 0; j < C2; ++j)
      for (int i = 0; i < R; ++i) {
        T acc = T(0);
        for (int k = 0; k < C; ++k) acc += (*this)(i, k) * o(k, j);
        out(i, j) = acc;
      }
    return out;
  }

  bool operator==(const Matrix& o) const { return std::equal(v_, v_ + R * C, o.v_); }
  bool operator!=(const Matrix& o) const { return !(*this == o); }

  Matrix<T, C, R> transpose() const {
    Matrix<T, C, R> t;
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < C; ++j) t(j, i) = (*this)(i, j);
    return t;
  }
  Matrix cwiseAbs() const { return map([](T a) { return static_cast<T>(std::abs(a)); }); }
  T maxCoeff() const { return *std::max_element(v_, v_ + R * C); }
  T minCoeff() const { return *std::min_element(v_, v_ + R * C); }
  T sum() const {
    T s = T(0);
    for (int i = 0; i < R * C; ++i) s += v_[i];
    return s;
  }
  T squaredNorm() const {
    T s = T(0);
    for (int i = 0; i < R * C; ++i) s += v_[i] * v_[i];
    return s;
  }
  T norm() const { return std::sqrt(squaredNorm()); }
  T dot(const Matrix& o) const {
    T s = T(0);
    for (int i = 0; i < R * C; ++i) s += v_[i] * o.v_[i];
    return s;
  }
  Matrix cross(const Matrix& o) const {
    static_assert(R * C == 3, "cross() needs 3-vectors");
    return Matrix(v_[1] * o.v_[2] - v_[2] * o.v_[1], v_[2] * o.v_[0] - v_[0] * o.v_[2],
                  v_[0] * o.v_[1] - v_[1] * o.v_[0]);
  }
  template <class U>
  Matrix<U, R, C> cast() const {
    Matrix<U, R, C> m;
    for (int i = 0; i < R * C; ++i) m.data()[i] = static_cast<U>(v_[i]);
    return m;
  }
  // by-value views (read) and writers (Eigen's segment<N>/block<N,M> lvalues)
  template <int N>
  Matrix<T, N, 1> segment(int start) const {
    Matrix<T, N, 1> s;
    for (int i = 0; i < N; ++i) s[i] = v_[start + i];
    return s;
  }
  template <int N>
  void setSegment(int start, const Matrix<T, N, 1>& s) {
    for (int i = 0; i < N; ++i) v_[start + i] = s[i];
  }
  template <int BR, int BC>
  Matrix<T, BR, BC> block(int r0, int c0) const {
    Matrix<T, BR, BC> b;
    for (int i = 0; i < BR; ++i)
      for (int j = 0; j < BC; ++j) b(i, j) = (*this)(r0 + i, c0 + j);
    return b;
  }

 private:
  template <class F>
  Matrix map(F f) const {
    Matrix m;
    for (int i = 0; i < R * C; ++i) m.v_[i] = f(v_[i]);
    return m;
  }
  template <class F>
  Matrix zip(const Matrix& o, F f) const {
    Matrix m;
    for (int i = 0; i < R * C; ++i) m.v_[i] = f(v_[i], o.v_[i]);
    return m;
  }
  T v_[R * C];
};

using Vec3 = Matrix<double, 3, 1>;
using Vec3i = Matrix<int, 3, 1>;
using Mat3 = Matrix<double, 3, 3>;
using Mat6 = Matrix<double, 6, 6>;

}  // namespace shellular
