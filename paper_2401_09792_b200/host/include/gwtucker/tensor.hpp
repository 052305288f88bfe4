// gwt:: drop-in API (B200 backend) — dense complex types and tensor operations.
// Mirrors /root/reference/proj/include/gwtucker/tensor.hpp (same names and
// semantics) without Eigen: Matrix/Vector provide the Eigen subset the
// reference API uses (column-major complex<double>).
#pragma once

#include <array>
#include <complex>
#include <cstddef>
#include <vector>

namespace gwt {

using Cplx = std::complex<double>;
using Index = std::ptrdiff_t;

class Matrix {
public:
    Matrix() = default;
    Matrix(Index rows, Index cols) : r_(rows), c_(cols), a_(static_cast<std::size_t>(rows * cols), Cplx(0, 0)) {}
    static Matrix Zero(Index rows, Index cols) { return Matrix(rows, cols); }
    static Matrix Identity(Index rows, Index cols);
    static Matrix Identity(Index n) { return Identity(n, n); }

    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    Cplx& operator()(Index i, Index j) { return a_[static_cast<std::size_t>(i + r_ * j)]; }
    const Cplx& operator()(Index i, Index j) const { return a_[static_cast<std::size_t>(i + r_ * j)]; }
    Cplx* data() { return a_.data(); }
    const Cplx* data() const { return a_.data(); }

    Matrix adjoint() const;
    Matrix transpose() const;
    Matrix conjugate() const;
    Matrix col(Index j) const;
    Matrix leftCols(Index n) const;
    void setCol(Index j, const Matrix& v);
    double squaredNorm() const;
    double norm() const;
    bool allFinite() const;

    Matrix operator*(const Matrix& o) const;
    Matrix operator+(const Matrix& o) const;
    Matrix operator-(const Matrix& o) const;
    Matrix& operator+=(const Matrix& o);
    Matrix& operator-=(const Matrix& o);
    friend Matrix operator*(const Cplx& s, const Matrix& m);
    friend Matrix operator*(double s, const Matrix& m) { return Cplx(s, 0.0) * m; }

protected:
    Index r_ = 0, c_ = 0;
    std::vector<Cplx> a_;
};

class Vector : public Matrix {
public:
    Vector() = default;
    explicit Vector(Index n) : Matrix(n, 1) {}
    Vector(const Matrix& m);  // column vector
    Cplx& operator()(Index i) { return a_[static_cast<std::size_t>(i)]; }
    const Cplx& operator()(Index i) const { return a_[static_cast<std::size_t>(i)]; }
    using Matrix::operator();
    void resize(Index n) { *this = Vector(n); }
};

using RealVector = std::vector<double>;

/// Dense complex 3-order tensor, mode-1-fastest: (i1,i2,i3) at i1 + d1*(i2 + d2*i3) (tensor.hpp:15-58).
class Tensor3 {
public:
    Tensor3() = default;
    Tensor3(int d1, int d2, int d3);
    int dim1() const { return d1_; }
    int dim2() const { return d2_; }
    int dim3() const { return d3_; }
    int dim(int mode) const;
    std::array<int, 3> dims() const { return {d1_, d2_, d3_}; }
    std::size_t size() const { return data_.size(); }
    Cplx& operator()(int i1, int i2, int i3) {
        return data_[static_cast<std::size_t>(i1) + static_cast<std::size_t>(d1_) * (i2 + static_cast<std::size_t>(d2_) * i3)];
    }
    const Cplx& operator()(int i1, int i2, int i3) const {
        return data_[static_cast<std::size_t>(i1) + static_cast<std::size_t>(d1_) * (i2 + static_cast<std::size_t>(d2_) * i3)];
    }
    const Cplx* data() const { return data_.data(); }
    Cplx* data() { return data_.data(); }
    Matrix mode1_view() const;   // copy (no Eigen::Map here)
    Matrix slice_view(int i3) const;
    bool same_dims(const Tensor3& o) const { return d1_ == o.d1_ && d2_ == o.d2_ && d3_ == o.d3_; }
    void setZero();

private:
    int d1_ = 0, d2_ = 0, d3_ = 0;
    std::vector<Cplx> data_;
};

Matrix matricize(const Tensor3& x, int mode);
Tensor3 dematricize(const Matrix& m, int mode, const std::array<int, 3>& dims);
/// Y = X x_mode U on the B200 (gwt_mode_product).
Tensor3 mode_product(const Tensor3& x, const Matrix& u, int mode);
/// M x N matrix with entry (i1,i2) = sum_i3 X(i1,i2,i3) * conj(c_(i3)) (B200 mode-3 product).
Matrix contract_mode3(const Tensor3& x, const Vector& coeff);
Cplx inner(const Tensor3& x, const Tensor3& y);
double squared_norm(const Tensor3& x);
double frobenius_norm(const Tensor3& x);

}  // namespace gwt
