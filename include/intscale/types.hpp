// B200 drop-in for proj/include/intscale/types.hpp (types.hpp:14-67).
// Eigen-free: a small owning row-major Dense<T> with the subset of the Eigen
// surface the reference API uses (rows, cols, size, data, operator(), resize,
// ==, Zero/Constant/Ones, minCoeff/maxCoeff), and the same exception taxonomy.
#pragma once

#include <algorithm>
#include <cstdint>
#include <initializer_list>
#include <stdexcept>
#include <string>
#include <vector>

namespace intscale {

using Index = std::int64_t;

template <class Scalar>
class Dense {
 public:
  Dense() = default;
  Dense(Index rows, Index cols) { resize(rows, cols); }
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index size() const { return rows_ * cols_; }
  Scalar* data() { return v_.data(); }
  const Scalar* data() const { return v_.data(); }
  void resize(Index rows, Index cols) {
    rows_ = rows;
    cols_ = cols;
    v_.assign(static_cast<std::size_t>(rows * cols), Scalar{});
  }
  Scalar& operator()(Index r, Index c) { return v_[static_cast<std::size_t>(r * cols_ + c)]; }
  const Scalar& operator()(Index r, Index c) const {
    return v_[static_cast<std::size_t>(r * cols_ + c)];
  }
  // Vector-style access (column vectors, rows x 1)
  Scalar& operator[](Index i) { return v_[static_cast<std::size_t>(i)]; }
  const Scalar& operator[](Index i) const { return v_[static_cast<std::size_t>(i)]; }
  Scalar minCoeff() const { return *std::min_element(v_.begin(), v_.end()); }
  Scalar maxCoeff() const { return *std::max_element(v_.begin(), v_.end()); }
  bool operator==(const Dense& o) const {
    return rows_ == o.rows_ && cols_ == o.cols_ && v_ == o.v_;
  }
  bool operator!=(const Dense& o) const { return !(*this == o); }
  static Dense Constant(Index rows, Index cols, Scalar v) {
    Dense d(rows, cols);
    std::fill(d.v_.begin(), d.v_.end(), v);
    return d;
  }
  static Dense Zero(Index rows, Index cols) { return Constant(rows, cols, Scalar{}); }
  static Dense Ones(Index rows, Index cols) { return Constant(rows, cols, Scalar(1)); }

 private:
  Index rows_ = 0, cols_ = 0;
  std::vector<Scalar> v_;
};

// Column vectors (Eigen::VectorXd / VectorXi stand-ins).
template <class Scalar>
class Vec : public Dense<Scalar> {
 public:
  Vec() = default;
  explicit Vec(Index n) : Dense<Scalar>(n, 1) {}
  Vec(std::initializer_list<Scalar> il) : Dense<Scalar>(static_cast<Index>(il.size()), 1) {
    Index i = 0;
    for (Scalar s : il) (*this)[i++] = s;
  }
  Index size() const { return this->rows(); }
  void resize(Index n) { Dense<Scalar>::resize(n, 1); }
  static Vec Constant(Index n, Scalar v) {
    Vec x(n);
    for (Index i = 0; i < n; ++i) x[i] = v;
    return x;
  }
  static Vec Zero(Index n) { return Constant(n, Scalar{}); }
  static Vec Ones(Index n) { return Constant(n, Scalar(1)); }
};

using MatF = Dense<float>;
using MatD = Dense<double>;
using MatQ = Dense<std::int16_t>;  // quantized codes, int16 for every bit width (types.hpp:19-21)
using MatI64 = Dense<std::int64_t>;
using VecD = Vec<double>;
using VecI = Vec<std::int32_t>;

// Exception hierarchy of types.hpp:29-67.
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct FormatError : Error {
  using Error::Error;
};
struct LengthError : Error {
  using Error::Error;
};
struct ValueError : Error {
  using Error::Error;
};
struct DimensionError : Error {
  using Error::Error;
};
struct ParamError : Error {
  using Error::Error;
};
struct OverflowError : Error {
  using Error::Error;
};
struct IoError : Error {
  using Error::Error;
};

}  // namespace intscale
