// PartialPivLU and the sparse subset of the Eigen shim (see shim.hpp) —
// TEST INFRASTRUCTURE ONLY.
#pragma once

#include "shim.hpp"

#include <utility>

namespace Eigen {

// Dense LU with row partial pivoting, P A = L U (unit L), as Eigen's
// PartialPivLU: the pivot of column k is the FIRST row of maximal |a| in k..n-1.
template <typename M>
class PartialPivLU {
  public:
    PartialPivLU() = default;
    template <typename A>
    explicit PartialPivLU(const A& a) {
        compute(a);
    }
    template <typename A>
    PartialPivLU& compute(const A& a_in) {
        lu_ = MatrixXd(a_in);
        n_ = lu_.rows();
        if (lu_.cols() != n_) throw std::logic_error("shim: PartialPivLU of a non-square matrix");
        perm_.resize((size_t)n_);
        for (Index i = 0; i < n_; ++i) perm_[(size_t)i] = i;
        l1_ = 0.0;
        for (Index j = 0; j < n_; ++j) {
            double s = 0.0;
            for (Index i = 0; i < n_; ++i) s += std::abs(lu_(i, j));
            l1_ = std::max(l1_, s);
        }
        for (Index k = 0; k < n_; ++k) {
            Index p = k;
            double best = std::abs(lu_(k, k));
            for (Index i = k + 1; i < n_; ++i)
                if (std::abs(lu_(i, k)) > best) {
                    best = std::abs(lu_(i, k));
                    p = i;
                }
            if (p != k) {
                for (Index j = 0; j < n_; ++j) std::swap(lu_(k, j), lu_(p, j));
                std::swap(perm_[(size_t)k], perm_[(size_t)p]);
            }
            const double piv = lu_(k, k);
            if (piv != 0.0)
                for (Index i = k + 1; i < n_; ++i) lu_(i, k) /= piv;
            for (Index j = k + 1; j < n_; ++j)
                for (Index i = k + 1; i < n_; ++i) lu_(i, j) -= lu_(i, k) * lu_(k, j);
        }
        return *this;
    }
    // x = A^-1 b for every column of b
    template <typename B>
    MatrixXd solve(const B& b_in) const {
        const MatrixXd b = MatrixXd(b_in);
        const bool row = b.rows() == 1 && b.cols() == n_ && n_ != 1;
        const Index nr = row ? n_ : b.rows(), nc = row ? 1 : b.cols();
        if (nr != n_) throw std::logic_error("shim: solve size mismatch");
        MatrixXd x(n_, nc);
        for (Index c = 0; c < nc; ++c) {
            for (Index i = 0; i < n_; ++i) x(i, c) = row ? b[perm_[(size_t)i]] : b(perm_[(size_t)i], c);
            for (Index i = 0; i < n_; ++i)
                for (Index k = 0; k < i; ++k) x(i, c) -= lu_(i, k) * x(k, c);
            for (Index i = n_ - 1; i >= 0; --i) {
                for (Index k = i + 1; k < n_; ++k) x(i, c) -= lu_(i, k) * x(k, c);
                x(i, c) /= lu_(i, i);
            }
        }
        return x;
    }
    // 1 / (||A||_1 ||A^-1||_1), exact (Eigen: the estimator of the same quantity)
    double rcond() const {
        if (n_ == 0) return 1.0;
        for (Index i = 0; i < n_; ++i)
            if (lu_(i, i) == 0.0) return 0.0;
        const MatrixXd inv = solve(MatrixXd::Identity(n_, n_));
        double ninv = 0.0;
        for (Index j = 0; j < n_; ++j) {
            double s = 0.0;
            for (Index i = 0; i < n_; ++i) s += std::abs(inv(i, j));
            ninv = std::max(ninv, s);
        }
        if (!std::isfinite(ninv) || l1_ == 0.0) return 0.0;
        return 1.0 / (l1_ * ninv);
    }
    const MatrixXd& matrixLU() const { return lu_; }

  private:
    MatrixXd lu_;
    std::vector<Index> perm_;
    Index n_ = 0;
    double l1_ = 0.0;
};

template <typename S, int R, int C, int Opt, int MR, int MC>
PartialPivLU<MatrixXd> Matrix<S, R, C, Opt, MR, MC>::partialPivLu() const {
    return PartialPivLU<MatrixXd>(*this);
}

template <typename T>
struct Triplet {
    Triplet(Index r, Index c, T v) : r_(r), c_(c), v_(v) {}
    Index row() const { return r_; }
    Index col() const { return c_; }
    T value() const { return v_; }
    Index r_, c_;
    T v_;
};

// Sparse matrix held dense (the direct-oracle systems pinned here are small).
template <typename T>
class SparseMatrix {
  public:
    SparseMatrix(Index rows, Index cols) : a_(rows, cols) {}
    template <typename It>
    void setFromTriplets(It first, It last) {
        a_.setZero();
        for (It it = first; it != last; ++it) a_(it->row(), it->col()) += it->value();   // duplicates summed
    }
    Index rows() const { return a_.rows(); }
    Index cols() const { return a_.cols(); }
    const MatrixXd& dense() const { return a_; }

  private:
    MatrixXd a_;
};

template <typename SM>
class SparseLU {
  public:
    void compute(const SM& a) {
        lu_.compute(a.dense());
        info_ = Success;
        const MatrixXd& f = lu_.matrixLU();
        for (Index i = 0; i < f.rows(); ++i)
            if (f(i, i) == 0.0 || !std::isfinite(f(i, i))) info_ = NumericalIssue;
    }
    template <typename B>
    VectorXd solve(const B& b) const {
        return VectorXd(lu_.solve(b));
    }
    ComputationInfo info() const { return info_; }

  private:
    PartialPivLU<MatrixXd> lu_;
    ComputationInfo info_ = NumericalIssue;
};

}  // namespace Eigen
