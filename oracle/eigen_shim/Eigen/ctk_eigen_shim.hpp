// TEST INFRASTRUCTURE ONLY (oracle/_ref build).  Eigen is an un-vendored dependency of
// the reference (CMakeLists.txt:12, "Eigen3 3.3 REQUIRED", no pinned version) and is
// absent from this image.  This is the smallest subset of Eigen 3.x's published API
// that lets the reference's hybrid.hpp / regparam.hpp / gmres.hpp / tv.hpp compile
// UNMODIFIED: dense MatrixXd/VectorXd, products, norms, a thin JacobiSVD (one-sided
// Hestenes-Jacobi, singular values sorted descending as Eigen documents) and a
// least-squares colPivHouseholderQr().solve() stand-in.  Results agree with Eigen's to
// rounding level, not bitwise; DESIGN.md records this.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <numeric>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;

enum DecompositionOptions { ComputeFullU = 4, ComputeThinU = 8, ComputeFullV = 16, ComputeThinV = 32 };

class VectorXd {
  public:
    VectorXd() = default;
    explicit VectorXd(Index n) : d_(std::size_t(n), 0.0) {}
    static VectorXd Zero(Index n) { return VectorXd(n); }
    static VectorXd Ones(Index n) {
        VectorXd v(n);
        std::fill(v.d_.begin(), v.d_.end(), 1.0);
        return v;
    }
    Index size() const { return Index(d_.size()); }
    Index rows() const { return size(); }
    double& operator()(Index i) { return d_[std::size_t(i)]; }
    double operator()(Index i) const { return d_[std::size_t(i)]; }
    double& operator[](Index i) { return d_[std::size_t(i)]; }
    double operator[](Index i) const { return d_[std::size_t(i)]; }
    double squaredNorm() const {
        double s = 0.0;
        for (double v : d_) s += v * v;
        return s;
    }
    double norm() const { return std::sqrt(squaredNorm()); }
    double dot(const VectorXd& o) const {
        double s = 0.0;
        for (std::size_t i = 0; i < d_.size(); ++i) s += d_[i] * o.d_[i];
        return s;
    }
    bool allFinite() const {
        for (double v : d_)
            if (!std::isfinite(v)) return false;
        return true;
    }
    VectorXd operator-(const VectorXd& o) const {
        VectorXd r(size());
        for (std::size_t i = 0; i < d_.size(); ++i) r.d_[i] = d_[i] - o.d_[i];
        return r;
    }
    VectorXd operator+(const VectorXd& o) const {
        VectorXd r(size());
        for (std::size_t i = 0; i < d_.size(); ++i) r.d_[i] = d_[i] + o.d_[i];
        return r;
    }
    VectorXd operator*(double s) const {
        VectorXd r(size());
        for (std::size_t i = 0; i < d_.size(); ++i) r.d_[i] = d_[i] * s;
        return r;
    }

  private:
    std::vector<double> d_;
};

inline VectorXd operator*(double s, const VectorXd& v) { return v * s; }

class MatrixXd;
template <class M>
class JacobiSVD;
class LeastSquaresSolve;

class MatrixXd {
  public:
    MatrixXd() = default;
    MatrixXd(Index r, Index c) : r_(r), c_(c), d_(std::size_t(r * c), 0.0) {}
    static MatrixXd Zero(Index r, Index c) { return MatrixXd(r, c); }
    static MatrixXd Identity(Index r, Index c) {
        MatrixXd m(r, c);
        for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
        return m;
    }
    Index rows() const { return r_; }
    Index cols() const { return c_; }
    double& operator()(Index i, Index j) { return d_[std::size_t(i * c_ + j)]; }
    double operator()(Index i, Index j) const { return d_[std::size_t(i * c_ + j)]; }
    MatrixXd transpose() const {
        MatrixXd t(c_, r_);
        for (Index i = 0; i < r_; ++i)
            for (Index j = 0; j < c_; ++j) t(j, i) = (*this)(i, j);
        return t;
    }
    bool allFinite() const {
        for (double v : d_)
            if (!std::isfinite(v)) return false;
        return true;
    }
    VectorXd operator*(const VectorXd& v) const {
        VectorXd r(r_);
        for (Index i = 0; i < r_; ++i) {
            double s = 0.0;
            for (Index j = 0; j < c_; ++j) s += (*this)(i, j) * v(j);
            r(i) = s;
        }
        return r;
    }
    MatrixXd operator*(const MatrixXd& o) const {
        MatrixXd r(r_, o.c_);
        for (Index i = 0; i < r_; ++i)
            for (Index j = 0; j < o.c_; ++j) {
                double s = 0.0;
                for (Index k = 0; k < c_; ++k) s += (*this)(i, k) * o(k, j);
                r(i, j) = s;
            }
        return r;
    }
    MatrixXd operator-(const MatrixXd& o) const {
        MatrixXd r(r_, c_);
        for (std::size_t i = 0; i < d_.size(); ++i) r.d_[i] = d_[i] - o.d_[i];
        return r;
    }
    inline LeastSquaresSolve colPivHouseholderQr() const;

  private:
    Index r_ = 0, c_ = 0;
    std::vector<double> d_;
};

// Thin SVD by one-sided (Hestenes) Jacobi rotations on the columns.
template <class M>
class JacobiSVD {
  public:
    JacobiSVD(const MatrixXd& a, int /*options*/) { compute(a); }
    const VectorXd& singularValues() const { return s_; }
    const MatrixXd& matrixU() const { return u_; }
    const MatrixXd& matrixV() const { return v_; }

  private:
    void compute(const MatrixXd& a0) {
        const bool tr = a0.rows() < a0.cols();
        MatrixXd a = tr ? a0.transpose() : a0;
        const Index m = a.rows(), n = a.cols();
        MatrixXd v = MatrixXd::Identity(n, n);
        for (int sweep = 0; sweep < 80; ++sweep) {
            double off = 0.0;
            for (Index p = 0; p < n - 1; ++p)
                for (Index q = p + 1; q < n; ++q) {
                    double alpha = 0, beta = 0, gamma = 0;
                    for (Index i = 0; i < m; ++i) {
                        alpha += a(i, p) * a(i, p);
                        beta += a(i, q) * a(i, q);
                        gamma += a(i, p) * a(i, q);
                    }
                    if (gamma == 0.0 || std::abs(gamma) <= 1e-300) continue;
                    const double rel = std::abs(gamma) / std::sqrt(alpha * beta);
                    off = std::max(off, rel);
                    if (rel < 1e-15) continue;
                    const double zeta = (beta - alpha) / (2.0 * gamma);
                    const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
                    const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
                    for (Index i = 0; i < m; ++i) {
                        const double x = a(i, p), y = a(i, q);
                        a(i, p) = c * x - s * y;
                        a(i, q) = s * x + c * y;
                    }
                    for (Index i = 0; i < n; ++i) {
                        const double x = v(i, p), y = v(i, q);
                        v(i, p) = c * x - s * y;
                        v(i, q) = s * x + c * y;
                    }
                }
            if (off < 1e-15) break;
        }
        std::vector<double> sig(static_cast<std::size_t>(n));
        for (Index j = 0; j < n; ++j) {
            double s = 0;
            for (Index i = 0; i < m; ++i) s += a(i, j) * a(i, j);
            sig[std::size_t(j)] = std::sqrt(s);
        }
        std::vector<Index> order(static_cast<std::size_t>(n));
        std::iota(order.begin(), order.end(), Index(0));
        std::stable_sort(order.begin(), order.end(),
                         [&](Index x, Index y) { return sig[std::size_t(x)] > sig[std::size_t(y)]; });
        MatrixXd u(m, n), vv(n, n);
        VectorXd s(n);
        for (Index jj = 0; jj < n; ++jj) {
            const Index j = order[std::size_t(jj)];
            s(jj) = sig[std::size_t(j)];
            for (Index i = 0; i < m; ++i) u(i, jj) = s(jj) > 0 ? a(i, j) / s(jj) : 0.0;
            for (Index i = 0; i < n; ++i) vv(i, jj) = v(i, j);
        }
        s_ = s;
        if (tr) {
            u_ = vv;
            v_ = u;
        } else {
            u_ = u;
            v_ = vv;
        }
    }
    VectorXd s_;
    MatrixXd u_, v_;
};

// colPivHouseholderQr().solve(b) stand-in: minimum-norm least-squares solution via the
// thin SVD (used only by gmres.hpp's projected_ls).
class LeastSquaresSolve {
  public:
    explicit LeastSquaresSolve(const MatrixXd& a) : a_(a) {}
    VectorXd solve(const VectorXd& b) const {
        JacobiSVD<MatrixXd> svd(a_, ComputeThinU | ComputeThinV);
        const VectorXd& s = svd.singularValues();
        VectorXd c = svd.matrixU().transpose() * b;
        const double tol = s.size() ? s(0) * 1e-13 : 0.0;
        VectorXd y(s.size());
        for (Index i = 0; i < s.size(); ++i) y(i) = s(i) > tol ? c(i) / s(i) : 0.0;
        return svd.matrixV() * y;
    }

  private:
    MatrixXd a_;
};

inline LeastSquaresSolve MatrixXd::colPivHouseholderQr() const { return LeastSquaresSolve(*this); }

}  // namespace Eigen
