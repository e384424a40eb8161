// exflow/matrix.hpp -- minimal dense matrix standing in for the Eigen types of
// the reference API (Eigen is not part of this build). Storage is ROW-MAJOR
// (the reference CountMatrix / MatrixXi are Eigen column-major); element
// access m(i, j), rows(), cols(), size(), sum() and equality keep the idioms
// reference callers use (e.g. counts.matrices[j](a, b), proj/src/trace.cpp:207).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <vector>

namespace exflow {

template <class T>
class Matrix {
  public:
    Matrix() = default;
    Matrix(std::int64_t rows, std::int64_t cols, T fill = T{})
        : rows_(rows), cols_(cols), data_(static_cast<std::size_t>(rows * cols), fill) {}

    static Matrix Zero(std::int64_t rows, std::int64_t cols) { return Matrix(rows, cols); }

    void resize(std::int64_t rows, std::int64_t cols) {
        rows_ = rows;
        cols_ = cols;
        data_.assign(static_cast<std::size_t>(rows * cols), T{});
    }

    T& operator()(std::int64_t i, std::int64_t j) { return data_[i * cols_ + j]; }
    const T& operator()(std::int64_t i, std::int64_t j) const { return data_[i * cols_ + j]; }

    std::int64_t rows() const { return rows_; }
    std::int64_t cols() const { return cols_; }
    std::int64_t size() const { return rows_ * cols_; }

    T* data() { return data_.data(); }
    const T* data() const { return data_.data(); }
    T* row_ptr(std::int64_t i) { return data_.data() + i * cols_; }
    const T* row_ptr(std::int64_t i) const { return data_.data() + i * cols_; }

    T sum() const {
        T s{};
        for (const T& v : data_) s += v;
        return s;
    }
    std::vector<T> rowwise_sum() const {
        std::vector<T> out(static_cast<std::size_t>(rows_), T{});
        for (std::int64_t i = 0; i < rows_; ++i)
            for (std::int64_t j = 0; j < cols_; ++j) out[i] += (*this)(i, j);
        return out;
    }

    bool operator==(const Matrix& o) const {
        return rows_ == o.rows_ && cols_ == o.cols_ && data_ == o.data_;
    }
    bool operator!=(const Matrix& o) const { return !(*this == o); }

  private:
    std::int64_t rows_ = 0;
    std::int64_t cols_ = 0;
    std::vector<T> data_;
};

}  // namespace exflow
