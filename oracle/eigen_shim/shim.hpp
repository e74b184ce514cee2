// Minimal Eigen-subset shim — TEST INFRASTRUCTURE ONLY (the oracle/_ref recipe).
//
// The reference (/root/reference/proj/include/hosweep/*.hpp) includes Eigen 3.3+,
// which is absent from this image.  This header provides exactly the subset of
// the Eigen API those headers use (quadrature, basis, mesh, assembly, romberg,
// sweepgraph, solver) so that the reference's OWN sources compile and run
// unmodified; oracle/ref_driver.cpp drives them to pin the oracle and the
// product (oracle/Makefile target `ref`, output in oracle/_ref/).  It is an
// original, eager implementation (no expression templates):
//   * Matrix<double, R, C, Options>: dynamic storage in either order, fixed
//     2-vectors / 2x2 matrices; every operator returns a column-major MatrixXd,
//     which converts implicitly to any other shape (like Eigen expressions);
//   * segment / row write-through proxies, Map (copying), transpose,
//     asDiagonal, cwise ops, norms, 2x2 inverse / determinant;
//   * PartialPivLU: row pivoting on the first max |a| of the column (as Eigen's
//     partial_lu), solve with vector or matrix right-hand sides, and rcond() =
//     1 / (||A||_1 ||A^-1||_1) computed EXACTLY (Eigen returns the Hager/Higham
//     estimate of the same quantity; it only feeds the > 1e-14 test);
//   * SparseMatrix / Triplet (duplicates summed) and SparseLU, the latter as a
//     dense partial-pivot LU (the direct-oracle problems pinned here are small).
// Products sum in ascending index order; Eigen's blocked GEMM sums in another
// order, so results agree with a real-Eigen build to round-off, not bitwise.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <stdexcept>
#include <type_traits>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
constexpr int Infinity = -1;
enum StorageOptions { ColMajor = 0, RowMajor = 1 };
enum ComputationInfo { Success = 0, NumericalIssue = 1 };

template <typename S, int R, int C, int Opt = ColMajor, int MR = R, int MC = C>
class Matrix;
using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;
using MatrixX2d = Matrix<double, Dynamic, 2>;
using Matrix2d = Matrix<double, 2, 2>;
using Vector2d = Matrix<double, 2, 1>;

template <typename M>
class SegmentRef;
template <typename M>
class RowRef;
template <typename M>
class PartialPivLU;

class DiagonalWrapper {
  public:
    explicit DiagonalWrapper(std::vector<double> d) : d_(std::move(d)) {}
    double operator[](Index i) const { return d_[(size_t)i]; }
  private:
    std::vector<double> d_;
};

template <typename S, int R, int C, int Opt, int MR, int MC>
class Matrix {
    static_assert(std::is_same<S, double>::value, "double only");

  public:
    using Scalar = double;

    Matrix() : r_(R > 0 ? R : 0), c_(C > 0 ? C : 0), v_((size_t)(r_ * c_), 0.0) {}
    template <typename I, typename = typename std::enable_if<std::is_integral<I>::value>::type>
    explicit Matrix(I n) : Matrix() {
        resize((Index)n);
    }
    template <typename I, typename J,
              typename = typename std::enable_if<std::is_integral<I>::value && std::is_integral<J>::value>::type>
    Matrix(I rows, J cols) : Matrix() {
        resize((Index)rows, (Index)cols);
    }
    Matrix(double x, double y) : Matrix() {   // Vector2d(x, y)
        static_assert(R == 2 && C == 1, "coordinate constructor: Vector2d only");
        v_[0] = x;
        v_[1] = y;
    }
    Matrix(const Matrix&) = default;
    Matrix(Matrix&&) = default;
    template <int R2, int C2, int O2, int A2, int B2>
    Matrix(const Matrix<double, R2, C2, O2, A2, B2>& o) : Matrix() {   // NOLINT: implicit, like Eigen
        assign(o);
    }
    template <typename M>
    Matrix(const SegmentRef<M>& s) : Matrix() {   // NOLINT
        assign(s.eval());
    }
    Matrix& operator=(const Matrix&) = default;
    Matrix& operator=(Matrix&&) = default;
    template <int R2, int C2, int O2, int A2, int B2>
    Matrix& operator=(const Matrix<double, R2, C2, O2, A2, B2>& o) {
        assign(o);
        return *this;
    }
    template <typename M>
    Matrix& operator=(const SegmentRef<M>& s) {
        assign(s.eval());
        return *this;
    }

    // ---- sizes and access
    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    double& operator()(Index i, Index j) { return v_[at(i, j)]; }
    double operator()(Index i, Index j) const { return v_[at(i, j)]; }
    double& operator()(Index i) { return v_[(size_t)i]; }
    double operator()(Index i) const { return v_[(size_t)i]; }
    double& operator[](Index i) { return v_[(size_t)i]; }
    double operator[](Index i) const { return v_[(size_t)i]; }

    void resize(Index n) {
        if (C == 1) resize(n, 1);
        else if (R == 1) resize(1, n);
        else throw std::logic_error("shim: resize(n) on a matrix");
    }
    void resize(Index rr, Index cc) {
        if ((R > 0 && rr != R) || (C > 0 && cc != C)) throw std::logic_error("shim: fixed-size resize");
        if (rr == r_ && cc == c_) return;
        r_ = rr;
        c_ = cc;
        v_.assign((size_t)(rr * cc), 0.0);
    }
    Matrix& setZero() {
        std::fill(v_.begin(), v_.end(), 0.0);
        return *this;
    }
    Matrix& setOnes() {
        std::fill(v_.begin(), v_.end(), 1.0);
        return *this;
    }
    static Matrix Zero() { return Matrix(); }
    static Matrix Zero(Index n) {
        Matrix m;
        m.resize(n);
        return m;
    }
    static Matrix Zero(Index rr, Index cc) {
        Matrix m;
        m.resize(rr, cc);
        return m;
    }
    static Matrix Ones(Index n) { return Zero(n).setOnes(); }
    static Matrix Ones(Index rr, Index cc) { return Zero(rr, cc).setOnes(); }
    static Matrix Identity(Index rr, Index cc) {
        Matrix m = Zero(rr, cc);
        for (Index i = 0; i < std::min(rr, cc); ++i) m(i, i) = 1.0;
        return m;
    }

    // ---- views (non-const: write-through proxies; const: copies)
    SegmentRef<Matrix> segment(Index s, Index n) { return SegmentRef<Matrix>(*this, s, n); }
    VectorXd segment(Index s, Index n) const {
        VectorXd out(n);
        for (Index i = 0; i < n; ++i) out[i] = v_[(size_t)(s + i)];
        return out;
    }
    RowRef<Matrix> row(Index i) { return RowRef<Matrix>(*this, i); }
    MatrixXd row(Index i) const {
        MatrixXd d(1, c_);
        for (Index j = 0; j < c_; ++j) d(0, j) = (*this)(i, j);
        return d;
    }
    VectorXd col(Index j) const {
        VectorXd out(r_);
        for (Index i = 0; i < r_; ++i) out[i] = (*this)(i, j);
        return out;
    }
    MatrixXd block(Index i0, Index j0, Index nr, Index nc) const {
        MatrixXd d(nr, nc);
        for (Index j = 0; j < nc; ++j)
            for (Index i = 0; i < nr; ++i) d(i, j) = (*this)(i0 + i, j0 + j);
        return d;
    }
    Matrix& noalias() { return *this; }

    MatrixXd transpose() const {
        MatrixXd d(c_, r_);
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) d(j, i) = (*this)(i, j);
        return d;
    }
    DiagonalWrapper asDiagonal() const { return DiagonalWrapper(linear()); }

    // ---- cwise / reductions
    MatrixXd cwiseAbs() const {
        MatrixXd d = *this;
        for (Index k = 0; k < d.size(); ++k) d[k] = std::abs(d[k]);
        return d;
    }
    template <int R2, int C2, int O2, int A2, int B2>
    MatrixXd cwiseProduct(const Matrix<double, R2, C2, O2, A2, B2>& o) const {
        MatrixXd d = *this;
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) d(i, j) *= o(i, j);
        return d;
    }
    double sum() const {
        double s = 0.0;
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) s += (*this)(i, j);
        return s;
    }
    template <int R2, int C2, int O2, int A2, int B2>
    double dot(const Matrix<double, R2, C2, O2, A2, B2>& o) const {
        if (o.size() != size()) throw std::logic_error("shim: dot size mismatch");
        double s = 0.0;
        for (Index k = 0; k < size(); ++k) s += v_[(size_t)k] * o[k];
        return s;
    }
    double squaredNorm() const { return dot(*this); }
    double norm() const { return std::sqrt(squaredNorm()); }
    void normalize() {
        const double n = norm();
        if (n > 0.0)
            for (double& x : v_) x /= n;
    }
    double maxCoeff() const { return *std::max_element(v_.begin(), v_.end()); }
    double minCoeff() const { return *std::min_element(v_.begin(), v_.end()); }
    template <int P>
    double lpNorm() const {
        static_assert(P == Infinity, "lpNorm<Infinity> only");
        double m = 0.0;
        for (double x : v_) m = std::max(m, std::abs(x));
        return m;
    }
    bool hasNaN() const {
        for (double x : v_)
            if (std::isnan(x)) return true;
        return false;
    }
    bool allFinite() const {
        for (double x : v_)
            if (!std::isfinite(x)) return false;
        return true;
    }
    double determinant() const {
        if (r_ != 2 || c_ != 2) throw std::logic_error("shim: determinant of 2x2 only");
        return (*this)(0, 0) * (*this)(1, 1) - (*this)(1, 0) * (*this)(0, 1);
    }
    MatrixXd inverse() const {
        if (r_ != 2 || c_ != 2) throw std::logic_error("shim: inverse of 2x2 only");
        // Eigen's compute_inverse<2x2>: multiply the adjugate by invdet = 1 / det
        // (LU/InverseImpl.h), and determinant() = m00 m11 - m10 m01 (Determinant.h)
        const double invdet = 1.0 / determinant();
        MatrixXd d(2, 2);
        d(0, 0) = (*this)(1, 1) * invdet;
        d(1, 0) = -(*this)(1, 0) * invdet;
        d(0, 1) = -(*this)(0, 1) * invdet;
        d(1, 1) = (*this)(0, 0) * invdet;
        return d;
    }
    PartialPivLU<MatrixXd> partialPivLu() const;

    // ---- compound assignment
    template <int R2, int C2, int O2, int A2, int B2>
    Matrix& operator+=(const Matrix<double, R2, C2, O2, A2, B2>& o) {
        same(o);
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) (*this)(i, j) += o(i, j);
        return *this;
    }
    template <int R2, int C2, int O2, int A2, int B2>
    Matrix& operator-=(const Matrix<double, R2, C2, O2, A2, B2>& o) {
        same(o);
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) (*this)(i, j) -= o(i, j);
        return *this;
    }
    Matrix& operator*=(double s) {
        for (double& x : v_) x *= s;
        return *this;
    }

    // values in column-major order
    std::vector<double> linear() const {
        std::vector<double> out((size_t)size());
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) out[(size_t)(j * r_ + i)] = (*this)(i, j);
        return out;
    }

  private:
    size_t at(Index i, Index j) const { return Opt == RowMajor ? (size_t)(i * c_ + j) : (size_t)(j * r_ + i); }
    template <typename M>
    void same(const M& o) const {
        // a vector accepts a vector-shaped operand of either orientation
        if (o.size() != size() || (o.rows() != r_ && !(std::min(r_, c_) == 1)))
            throw std::logic_error("shim: size mismatch");
    }
    template <int R2, int C2, int O2, int A2, int B2>
    void assign(const Matrix<double, R2, C2, O2, A2, B2>& o) {
        Index rr = o.rows(), cc = o.cols();
        const bool flip = (C == 1 && rr == 1 && cc != 1) || (R == 1 && cc == 1 && rr != 1);
        if (flip) std::swap(rr, cc);
        std::vector<double> tmp = o.linear();   // o may alias *this
        resize(rr, cc);
        for (Index j = 0; j < cc; ++j)
            for (Index i = 0; i < rr; ++i) (*this)(i, j) = tmp[(size_t)(j * rr + i)];
    }

    Index r_, c_;
    std::vector<double> v_;
};

// ---- free operators (results are column-major MatrixXd)
template <typename T>
struct is_mat : std::false_type {};
template <int R, int C, int O, int A, int B>
struct is_mat<Matrix<double, R, C, O, A, B>> : std::true_type {};
template <typename T>
using mat_t = typename std::enable_if<is_mat<T>::value || std::is_base_of<MatrixXd, T>::value, MatrixXd>::type;

template <typename A>
MatrixXd as_mat(const A& a) {
    return MatrixXd(a);
}

template <typename A, typename B>
mat_t<A> operator+(const A& a, const B& b) {
    MatrixXd x = as_mat(a);
    x += as_mat(b);
    return x;
}
template <typename A, typename B>
mat_t<A> operator-(const A& a, const B& b) {
    MatrixXd x = as_mat(a);
    x -= as_mat(b);
    return x;
}
template <typename A>
mat_t<A> operator-(const A& a) {
    MatrixXd x = as_mat(a);
    for (Index k = 0; k < x.size(); ++k) x[k] = -x[k];
    return x;
}
template <typename A>
mat_t<A> operator*(double s, const A& a) {
    MatrixXd x = as_mat(a);
    for (Index k = 0; k < x.size(); ++k) x[k] = s * x[k];
    return x;
}
template <typename A>
mat_t<A> operator*(const A& a, double s) {
    MatrixXd x = as_mat(a);
    for (Index k = 0; k < x.size(); ++k) x[k] = x[k] * s;
    return x;
}
template <typename A>
mat_t<A> operator/(const A& a, double s) {
    MatrixXd x = as_mat(a);
    for (Index k = 0; k < x.size(); ++k) x[k] = x[k] / s;
    return x;
}
// matrix product: k summed in ascending order
template <typename A, typename B>
typename std::enable_if<(is_mat<A>::value || std::is_base_of<MatrixXd, A>::value) &&
                            (is_mat<B>::value || std::is_base_of<MatrixXd, B>::value),
                        MatrixXd>::type
operator*(const A& a, const B& b) {
    const MatrixXd x = as_mat(a), y = as_mat(b);
    if (x.cols() != y.rows()) throw std::logic_error("shim: product size mismatch");
    MatrixXd z(x.rows(), y.cols());
    for (Index j = 0; j < y.cols(); ++j)
        for (Index i = 0; i < x.rows(); ++i) {
            double s = 0.0;
            for (Index k = 0; k < x.cols(); ++k) s += x(i, k) * y(k, j);
            z(i, j) = s;
        }
    return z;
}
template <typename A>
mat_t<A> operator*(const A& a, const DiagonalWrapper& d) {
    MatrixXd x = as_mat(a);
    for (Index j = 0; j < x.cols(); ++j)
        for (Index i = 0; i < x.rows(); ++i) x(i, j) *= d[j];
    return x;
}
template <typename A>
mat_t<A> operator*(const DiagonalWrapper& d, const A& a) {
    MatrixXd x = as_mat(a);
    for (Index j = 0; j < x.cols(); ++j)
        for (Index i = 0; i < x.rows(); ++i) x(i, j) *= d[i];
    return x;
}

// ---- write-through views
template <typename M>
class SegmentRef {
  public:
    SegmentRef(M& m, Index s, Index n) : m_(&m), s_(s), n_(n) {}
    Index size() const { return n_; }
    double& operator[](Index i) { return (*m_)[s_ + i]; }
    double operator[](Index i) const { return (*m_)[s_ + i]; }
    double& operator()(Index i) { return (*m_)[s_ + i]; }
    VectorXd eval() const {
        VectorXd d(n_);
        for (Index i = 0; i < n_; ++i) d[i] = (*m_)[s_ + i];
        return d;
    }
    SegmentRef& noalias() { return *this; }
    template <typename T>
    SegmentRef& operator=(const T& x) {
        const VectorXd d = VectorXd(x);
        if (d.size() != n_) throw std::logic_error("shim: segment = size mismatch");
        for (Index i = 0; i < n_; ++i) (*m_)[s_ + i] = d[i];
        return *this;
    }
    SegmentRef& operator=(const SegmentRef& o) { return operator= <VectorXd>(o.eval()); }
    template <typename T>
    SegmentRef& operator+=(const T& x) {
        const VectorXd d = VectorXd(x);
        if (d.size() != n_) throw std::logic_error("shim: segment += size mismatch");
        for (Index i = 0; i < n_; ++i) (*m_)[s_ + i] += d[i];
        return *this;
    }
    template <typename T>
    SegmentRef& operator-=(const T& x) {
        const VectorXd d = VectorXd(x);
        if (d.size() != n_) throw std::logic_error("shim: segment -= size mismatch");
        for (Index i = 0; i < n_; ++i) (*m_)[s_ + i] -= d[i];
        return *this;
    }
    double sum() const { return eval().sum(); }

  private:
    M* m_;
    Index s_, n_;
};

template <typename M>
class RowRef {
  public:
    RowRef(M& m, Index i) : m_(&m), i_(i) {}
    template <typename T>
    RowRef& operator=(const T& x) {
        const MatrixXd d = MatrixXd(x);
        if (d.size() != m_->cols()) throw std::logic_error("shim: row = size mismatch");
        for (Index j = 0; j < m_->cols(); ++j) (*m_)(i_, j) = d[j];
        return *this;
    }

  private:
    M* m_;
    Index i_;
};

// Map<const Matrix<...>>(ptr, rows, cols): a copy in the mapped storage order
template <typename T>
class Map : public MatrixXd {
  public:
    using Plain = typename std::remove_const<T>::type;
    Map(const double* p, Index rows, Index cols) : MatrixXd(rows, cols) {
        const bool row_major = IsRowMajor<Plain>::value;
        for (Index j = 0; j < cols; ++j)
            for (Index i = 0; i < rows; ++i) (*this)(i, j) = row_major ? p[i * cols + j] : p[j * rows + i];
    }

  private:
    template <typename X>
    struct IsRowMajor : std::false_type {};
    template <int R, int C, int A, int B>
    struct IsRowMajor<Matrix<double, R, C, RowMajor, A, B>> : std::true_type {};
};

}  // namespace Eigen
