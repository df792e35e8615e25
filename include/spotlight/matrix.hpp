// Drop-in for the container half of proj/include/spotlight/matrix.hpp: a
// dense row-major Matrix<T> with the same accessors, so code written against
// the reference compiles unchanged. matmul<T> (float / double) runs on the
// GPU (spl_matmul) with the reference build's per-output FMA order; the
// training-side products matmul_bt / add_matmul_at are not re-exposed.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <span>
#include <string>
#include <vector>

#include "spotlight/errors.hpp"

namespace spotlight {

template <typename T>
class Matrix {
public:
    Matrix() = default;
    Matrix(std::size_t rows, std::size_t cols) : r_(rows), c_(cols), v_(rows * cols, T(0)) {}
    Matrix(std::size_t rows, std::size_t cols, std::vector<T> values)
        : r_(rows), c_(cols), v_(std::move(values)) {
        if (v_.size() != r_ * c_)
            throw DimensionError("Matrix: data size " + std::to_string(v_.size()) +
                                 " does not match " + std::to_string(r_) + "x" + std::to_string(c_));
    }

    std::size_t rows() const { return r_; }
    std::size_t cols() const { return c_; }
    std::size_t size() const { return v_.size(); }
    bool empty() const { return v_.empty(); }

    T& operator()(std::size_t i, std::size_t j) { return v_[i * c_ + j]; }
    const T& operator()(std::size_t i, std::size_t j) const { return v_[i * c_ + j]; }

    std::span<T> row(std::size_t i) { return std::span<T>(v_.data() + i * c_, c_); }
    std::span<const T> row(std::size_t i) const { return std::span<const T>(v_.data() + i * c_, c_); }

    T* data() { return v_.data(); }
    const T* data() const { return v_.data(); }
    const std::vector<T>& values() const { return v_; }
    void fill(T x) { std::fill(v_.begin(), v_.end(), x); }

    bool all_finite() const {
        return std::all_of(v_.begin(), v_.end(),
                           [](const T& x) { return std::isfinite(static_cast<double>(x)); });
    }
    bool operator==(const Matrix& o) const { return r_ == o.r_ && c_ == o.c_ && v_ == o.v_; }

private:
    std::size_t r_ = 0, c_ = 0;
    std::vector<T> v_;
};

/// Sequential dot product and Euclidean norm (matrix.hpp:145-155): scalar
/// host helpers callers use on rows of a Matrix.
template <typename T>
T dot(std::span<const T> a, std::span<const T> b) {
    T acc = T(0);
    for (std::size_t i = 0; i < a.size(); ++i) acc += a[i] * b[i];
    return acc;
}

template <typename T>
T norm2(std::span<const T> a) {
    return std::sqrt(dot(a, a));
}

/// C = A * B (matrix.hpp:81-99): every output an FMA chain over the inner
/// index in order, as the reference's Release build computes it. GPU.
/// DimensionError("matmul: inner dimensions ... do not match").
template <typename T>
Matrix<T> matmul(const Matrix<T>& a, const Matrix<T>& b);
extern template Matrix<float> matmul<float>(const Matrix<float>&, const Matrix<float>&);
extern template Matrix<double> matmul<double>(const Matrix<double>&, const Matrix<double>&);

template <typename To, typename From>
Matrix<To> matrix_cast(const Matrix<From>& m) {
    std::vector<To> v(m.values().begin(), m.values().end());
    return Matrix<To>(m.rows(), m.cols(), std::move(v));
}

}  // namespace spotlight
