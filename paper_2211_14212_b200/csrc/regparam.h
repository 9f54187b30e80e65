// Host fp64 projected-problem helpers (regparam.cpp).
#pragma once
#include <vector>

#include "../../include/ctk_b200.h"

namespace ctkb {

// H is row-major (m x n), m >= n.  U: m x n, s: n (descending), V: n x n.
void thin_svd(const std::vector<double>& H, int m, int n, std::vector<double>& U, std::vector<double>& s,
              std::vector<double>& V);

struct ProjectedSvd {
    std::vector<double> sigma, rhs;
    double perp2 = 0.0;
    int k = 0;
    ProjectedSvd(const std::vector<double>& H, int k, double beta1);
    double discrepancy2(double lambda) const;
    double gcv(double lambda) const;
};

double dp_lambda(const std::vector<double>& H, int k, double beta1, double nl);
double gcv_lambda(const std::vector<double>& H, int k, double beta1);
std::vector<double> projected_tikhonov(const std::vector<double>& H, int k, double beta1, double lambda,
                                       double* fit_resid);
double choose_lambda(const ctk_hybrid_strategy& st, const std::vector<double>& H, int k, double beta1);
// min || beta1 e1 - H y || for the (k+1) x k Hessenberg of Arnoldi (gmres.hpp:24-31)
std::vector<double> projected_ls(const std::vector<double>& H, int k, double beta1, double* resid);

}  // namespace ctkb
