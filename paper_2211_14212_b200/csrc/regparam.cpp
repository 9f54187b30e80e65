// Host fp64 work on the (k+1) x k projected problem of hybrid LSQR -- O(k^3), not GPU
// work (SURVEY.md 2.1 "reg-param choice").  Restates, without Eigen:
//   ProjectedSvd / discrepancy2 / gcv   regparam.hpp:26-71
//   dp_lambda                           regparam.hpp:79-113
//   gcv_lambda                          regparam.hpp:114-159
//   projected_tikhonov                  hybrid.hpp:37-55
//   choose_lambda                       hybrid.hpp:57-72
// The thin SVD is a one-sided Jacobi (singular values descending, like Eigen's
// JacobiSVD); results agree with Eigen to rounding level.
#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <vector>

#include "ctk_internal.h"
#include "regparam.h"

namespace ctkb {

void thin_svd(const std::vector<double>& a0, int m, int n, std::vector<double>& U, std::vector<double>& s,
              std::vector<double>& V) {
    // requires m >= n (projected problems are (k+1) x k)
    std::vector<double> a = a0;  // row-major m x n, columns rotated in place
    V.assign(size_t(n) * n, 0.0);
    for (int i = 0; i < n; ++i) V[size_t(i) * n + i] = 1.0;
    for (int sweep = 0; sweep < 80; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                double alpha = 0, beta = 0, gamma = 0;
                for (int i = 0; i < m; ++i) {
                    const double x = a[size_t(i) * n + p], y = a[size_t(i) * n + q];
                    alpha += x * x;
                    beta += y * y;
                    gamma += x * y;
                }
                if (gamma == 0.0) continue;
                const double rel = std::abs(gamma) / std::sqrt(alpha * beta);
                off = std::max(off, rel);
                if (rel < 1e-15) continue;
                const double zeta = (beta - alpha) / (2.0 * gamma);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
                for (int i = 0; i < m; ++i) {
                    const double x = a[size_t(i) * n + p], y = a[size_t(i) * n + q];
                    a[size_t(i) * n + p] = c * x - sn * y;
                    a[size_t(i) * n + q] = sn * x + c * y;
                }
                for (int i = 0; i < n; ++i) {
                    const double x = V[size_t(i) * n + p], y = V[size_t(i) * n + q];
                    V[size_t(i) * n + p] = c * x - sn * y;
                    V[size_t(i) * n + q] = sn * x + c * y;
                }
            }
        if (off < 1e-15) break;
    }
    std::vector<double> sig(static_cast<size_t>(n));
    for (int j = 0; j < n; ++j) {
        double t = 0;
        for (int i = 0; i < m; ++i) t += a[size_t(i) * n + j] * a[size_t(i) * n + j];
        sig[size_t(j)] = std::sqrt(t);
    }
    std::vector<int> order(static_cast<size_t>(n));
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return sig[size_t(x)] > sig[size_t(y)]; });
    U.assign(size_t(m) * n, 0.0);
    s.assign(size_t(n), 0.0);
    std::vector<double> Vs(size_t(n) * n);
    for (int jj = 0; jj < n; ++jj) {
        const int j = order[size_t(jj)];
        s[size_t(jj)] = sig[size_t(j)];
        for (int i = 0; i < m; ++i) U[size_t(i) * n + jj] = sig[size_t(j)] > 0 ? a[size_t(i) * n + j] / sig[size_t(j)] : 0.0;
        for (int i = 0; i < n; ++i) Vs[size_t(i) * n + jj] = V[size_t(i) * n + j];
    }
    V.swap(Vs);
}

ProjectedSvd::ProjectedSvd(const std::vector<double>& H, int k, double beta1) : k(k) {
    for (double v : H)
        if (!std::isfinite(v)) fail(CTK_E_PARAMETER, "projected problem has non-finite entries");
    if (!std::isfinite(beta1)) fail(CTK_E_PARAMETER, "projected problem has non-finite entries");
    std::vector<double> U, V;
    thin_svd(H, k + 1, k, U, sigma, V);
    rhs.assign(size_t(k), 0.0);
    double sq = 0.0;
    for (int i = 0; i < k; ++i) {
        rhs[size_t(i)] = U[size_t(i)] * beta1;  // U^T (beta1 e1): first row of U
        sq += rhs[size_t(i)] * rhs[size_t(i)];
    }
    perp2 = std::max(0.0, beta1 * beta1 - sq);
}

double ProjectedSvd::discrepancy2(double lambda) const {
    const double l2 = lambda * lambda;
    double s = perp2;
    for (int i = 0; i < k; ++i) {
        const double d = sigma[size_t(i)] * sigma[size_t(i)] + l2;
        const double f = (d > 0.0) ? l2 / d : 1.0;
        s += (rhs[size_t(i)] * f) * (rhs[size_t(i)] * f);
    }
    return s;
}

double ProjectedSvd::gcv(double lambda) const {
    double num = perp2;
    double trace = double(k) + 1.0;
    for (int i = 0; i < k; ++i) {
        const double s2 = sigma[size_t(i)] * sigma[size_t(i)];
        const double r = lambda / (s2 + lambda);
        num += (rhs[size_t(i)] * r) * (rhs[size_t(i)] * r);
        trace -= s2 / (s2 + lambda);
    }
    return num / (trace * trace);
}

double dp_lambda(const std::vector<double>& H, int k, double beta1, double nl) {
    if (!(nl > 0.0 && nl < 1.0)) fail(CTK_E_PARAMETER, "noise level must lie in (0,1)");
    ProjectedSvd svd(H, k, beta1);
    const double target = nl * nl * beta1 * beta1;
    constexpr double rel_tol = 1e-6;
    if (svd.discrepancy2(0.0) >= target * (1.0 - 1e-12)) return 0.0;
    const double smax = svd.sigma[0];
    const double lo = 1e-10 * smax, hi = 1e10 * smax;
    if (svd.discrepancy2(lo) >= target) {
        double a = 0.0, b = lo;
        for (int it = 0; it < 200; ++it) {
            const double mid = 0.5 * (a + b);
            const double d = svd.discrepancy2(mid);
            if (std::abs(d - target) <= rel_tol * target) return mid;
            (d < target ? a : b) = mid;
        }
        return 0.5 * (a + b);
    }
    double llo = std::log(lo), lhi = std::log(hi);
    double mid = 0.5 * (llo + lhi);
    for (int it = 0; it < 60; ++it) {
        mid = 0.5 * (llo + lhi);
        const double d = svd.discrepancy2(std::exp(mid));
        if (std::abs(d - target) <= rel_tol * target) break;
        (d < target ? llo : lhi) = mid;
    }
    return std::exp(mid);
}

double gcv_lambda(const std::vector<double>& H, int k, double beta1) {
    ProjectedSvd svd(H, k, beta1);
    const double smax = svd.sigma[0];
    if (!(smax > 0.0)) fail(CTK_E_PARAMETER, "gcv_lambda: projected matrix is zero");
    const double lo = std::log(1e-10 * smax * smax);
    const double hi = std::log(1e10 * smax * smax);
    constexpr int scan_points = 1001;
    int best = 0;
    double best_val = std::numeric_limits<double>::infinity();
    for (int i = 0; i < scan_points; ++i) {
        const double ll = lo + (hi - lo) * i / (scan_points - 1);
        const double v = svd.gcv(std::exp(ll));
        if (v < best_val) {
            best_val = v;
            best = i;
        }
    }
    const double step = (hi - lo) / (scan_points - 1);
    double a = lo + step * std::max(0, best - 1);
    double b = lo + step * std::min(scan_points - 1, best + 1);
    constexpr double inv_phi = 0.6180339887498949;
    double c = b - inv_phi * (b - a);
    double d = a + inv_phi * (b - a);
    double fc = svd.gcv(std::exp(c)), fd = svd.gcv(std::exp(d));
    for (int it = 0; it < 200 && (b - a) > 1e-10; ++it) {
        if (fc < fd) {
            b = d;
            d = c;
            fd = fc;
            c = b - inv_phi * (b - a);
            fc = svd.gcv(std::exp(c));
        } else {
            a = c;
            c = d;
            fc = fd;
            d = a + inv_phi * (b - a);
            fd = svd.gcv(std::exp(d));
        }
    }
    return std::exp(0.5 * (a + b));
}

std::vector<double> projected_tikhonov(const std::vector<double>& H, int k, double beta1, double lambda,
                                       double* fit_resid) {
    std::vector<double> U, s, V;
    thin_svd(H, k + 1, k, U, s, V);
    std::vector<double> yf(static_cast<size_t>(k));
    for (int i = 0; i < k; ++i) {
        const double coef = U[size_t(i)] * beta1;  // (U^T rhs)_i, rhs = beta1 e1
        const double d = s[size_t(i)] * s[size_t(i)] + lambda * lambda;
        yf[size_t(i)] = (d > 0.0) ? s[size_t(i)] * coef / d : 0.0;
    }
    std::vector<double> y(size_t(k), 0.0);
    for (int r = 0; r < k; ++r) {
        double t = 0.0;
        for (int c = 0; c < k; ++c) t += V[size_t(r) * k + c] * yf[size_t(c)];
        y[size_t(r)] = t;
    }
    if (fit_resid) {
        double sq = 0.0;
        for (int r = 0; r < k + 1; ++r) {
            double t = (r == 0) ? beta1 : 0.0;
            for (int c = 0; c < k; ++c) t -= H[size_t(r) * k + c] * y[size_t(c)];
            sq += t * t;
        }
        *fit_resid = std::sqrt(sq);
    }
    return y;
}

double choose_lambda(const ctk_hybrid_strategy& st, const std::vector<double>& H, int k, double beta1) {
    switch (st.kind) {
        case CTK_LAMBDA_FIXED: return st.lambda;
        case CTK_LAMBDA_DP: return dp_lambda(H, k, beta1, st.noise_level);
        case CTK_LAMBDA_GCV: return std::sqrt(std::max(0.0, gcv_lambda(H, k, beta1)));
    }
    return 0.0;
}

// gmres.hpp:24-31 solves with Eigen's colPivHouseholderQr().  For full column rank (every
// Arnoldi step that did not break down) the least-squares solution is unique and this
// SVD-based solve agrees with it to rounding; a numerically rank-deficient H takes the
// minimum-norm solution over singular values above 1e-13 s_max.  The residual is formed
// explicitly as || rhs - H y || like the reference.
std::vector<double> projected_ls(const std::vector<double>& H, int k, double beta1, double* resid) {
    std::vector<double> U, s, V;
    thin_svd(H, k + 1, k, U, s, V);
    const double tol = k > 0 ? s[0] * 1e-13 : 0.0;
    std::vector<double> c(size_t(k), 0.0), y(size_t(k), 0.0);
    for (int i = 0; i < k; ++i) c[size_t(i)] = s[size_t(i)] > tol ? U[size_t(i)] * beta1 / s[size_t(i)] : 0.0;
    for (int r = 0; r < k; ++r) {
        double acc = 0.0;
        for (int i = 0; i < k; ++i) acc += V[size_t(r) * k + i] * c[size_t(i)];
        y[size_t(r)] = acc;
    }
    if (resid) {
        double sq = 0.0;
        for (int r = 0; r <= k; ++r) {
            double hy = 0.0;
            for (int j = 0; j < k; ++j) hy += H[size_t(r) * k + j] * y[size_t(j)];
            const double e = (r == 0 ? beta1 : 0.0) - hy;
            sq += e * e;
        }
        *resid = std::sqrt(sq);
    }
    return y;
}

}  // namespace ctkb
