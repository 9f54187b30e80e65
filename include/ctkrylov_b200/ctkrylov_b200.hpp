// ctkrylov_b200.hpp -- header-only C++ drop-in over the C-ABI (include/ctk_b200.h).
//
// Written against the reference's own types (ctk::ConeGeometry, ctk::OperatorPair<T>,
// ctk::SolverOptions<T>, ctk::SolveResult<T> from /root/reference/proj/include), so a C++
// user of the reference swaps
//     auto pair = ctk::projector_pair<T>(geom, variant);      // operators.hpp:91-115
//     auto res  = ctk::lsqr(pair, b, opts);                     // solvers.hpp:62-126
// for
//     auto pair = ctkb::projector_pair<T>(geom, variant);       // sm_100a Ax / A^T b
//     auto res  = ctkb::lsqr(pair, b, opts);                    // device-resident solver
// ctkb::projector_pair returns a ctk::OperatorPair<T> (subclass) whose host-span
// std::function callbacks (operators.hpp:18-45) run the B200 kernels, so the reference's
// own CPU solvers and wrappers (augment_tikhonov, stack_weighted_gradient) accept it
// unchanged.  Errors come back as the reference's exception types (types.hpp:14-31).
// Build: -I<reference>/proj/include -I<repo>/include, link libctk_b200.so.
#pragma once

#include <algorithm>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "ctkrylov/operators.hpp"
#include "ctkrylov/solve_log.hpp"
#include "../ctk_b200.h"

namespace ctkb {

[[noreturn]] inline void rethrow_status(int rc) {
    char msg[512];
    ctk_last_error(msg, sizeof msg);
    switch (rc) {
        case CTK_E_DIMENSION: throw ctk::DimensionError(msg);
        case CTK_E_GEOMETRY: throw ctk::GeometryError(msg);
        case CTK_E_PARAMETER: throw ctk::ParameterError(msg);
        case CTK_E_DEGENERATE: throw ctk::DegenerateInputError(msg);
        case CTK_E_NUMERICAL: throw ctk::NumericalError(msg, ctk_last_error_iteration());
        default: throw std::runtime_error(std::string("ctk_b200: ") + msg);
    }
}
inline void check(int rc) {
    if (rc != CTK_OK) rethrow_status(rc);
}

/// RAII owner of a native geometry handle (validated ConeGeometry + device tables).
class Handle {
  public:
    explicit Handle(const ctk::ConeGeometry& g) : angles_(g.angles) {
        ctk_geom_desc d{};
        d.mode = int(g.mode);
        d.source_to_origin = g.source_to_origin;
        d.origin_to_detector = g.origin_to_detector;
        d.detector_pixel_size = g.detector_pixel_size;
        d.nu = g.nu;
        d.nv = g.nv;
        d.nx = g.vol.nx;
        d.ny = g.vol.ny;
        d.nz = g.vol.nz;
        d.spacing = g.vol.spacing;
        d.n_angles = int(angles_.size());
        d.angles = angles_.data();
        check(ctk_geom_create(&d, &h_));
    }
    ~Handle() {
        if (h_) ctk_geom_destroy(h_);
    }
    Handle(const Handle&) = delete;
    Handle& operator=(const Handle&) = delete;
    ctk_geom* get() const { return h_; }

  private:
    std::vector<double> angles_;
    ctk_geom* h_ = nullptr;
};

template <class T>
struct Ops;
template <>
struct Ops<float> {
    static int ax(ctk_geom* g, const float* x, float* y) { return ctk_ax_host_f32(g, x, y); }
    static int atb(ctk_geom* g, int v, const float* y, float* x) { return ctk_atb_host_f32(g, v, y, x); }
    static int cgls(ctk_geom* g, int v, const float* b, const ctk_solver_opts* o, float* x, ctk_solve_log* l) { return ctk_cgls_f32(g, v, b, o, x, l); }
    static int lsqr(ctk_geom* g, int v, const float* b, const ctk_solver_opts* o, float* x, ctk_solve_log* l) { return ctk_lsqr_f32(g, v, b, o, x, l); }
    static int sirt(ctk_geom* g, int v, const float* b, const ctk_solver_opts* o, float* x, ctk_solve_log* l) { return ctk_sirt_f32(g, v, b, o, x, l); }
    static int ab_gmres(ctk_geom* g, int v, const float* b, const ctk_solver_opts* o, float* x, ctk_solve_log* l) { return ctk_ab_gmres_f32(g, v, b, o, x, l); }
    static int ba_gmres(ctk_geom* g, int v, const float* b, const ctk_solver_opts* o, float* x, ctk_solve_log* l) { return ctk_ba_gmres_f32(g, v, b, o, x, l); }
    static int lsmr(ctk_geom* g, int v, const float* b, double lam, const ctk_solver_opts* o, float* x, ctk_solve_log* l) { return ctk_lsmr_f32(g, v, b, lam, o, x, l); }
    static int hybrid(ctk_geom* g, int v, const float* b, const ctk_hybrid_strategy* s, const ctk_solver_opts* o, float* x, ctk_solve_log* l) { return ctk_hybrid_lsqr_f32(g, v, b, s, o, x, l); }
    static int flsqr_tv(ctk_geom* g, int v, const float* b, const ctk_hybrid_strategy* s, const ctk_solver_opts* o, float* x, ctk_solve_log* l) { return ctk_flsqr_tv_f32(g, v, b, s, o, x, l); }
    static int tv(ctk_geom* g, int v, const float* b, double lam, int oi, int ii, const ctk_solver_opts* o, int w, float* x, ctk_solve_log* l) { return ctk_cgls_tv_f32(g, v, b, lam, oi, ii, o, w, x, l); }
};
template <>
struct Ops<double> {
    static int ax(ctk_geom* g, const double* x, double* y) { return ctk_ax_host_f64(g, x, y); }
    static int atb(ctk_geom* g, int v, const double* y, double* x) { return ctk_atb_host_f64(g, v, y, x); }
    static int cgls(ctk_geom* g, int v, const double* b, const ctk_solver_opts* o, double* x, ctk_solve_log* l) { return ctk_cgls_f64(g, v, b, o, x, l); }
    static int lsqr(ctk_geom* g, int v, const double* b, const ctk_solver_opts* o, double* x, ctk_solve_log* l) { return ctk_lsqr_f64(g, v, b, o, x, l); }
    static int sirt(ctk_geom* g, int v, const double* b, const ctk_solver_opts* o, double* x, ctk_solve_log* l) { return ctk_sirt_f64(g, v, b, o, x, l); }
    static int ab_gmres(ctk_geom* g, int v, const double* b, const ctk_solver_opts* o, double* x, ctk_solve_log* l) { return ctk_ab_gmres_f64(g, v, b, o, x, l); }
    static int ba_gmres(ctk_geom* g, int v, const double* b, const ctk_solver_opts* o, double* x, ctk_solve_log* l) { return ctk_ba_gmres_f64(g, v, b, o, x, l); }
    static int lsmr(ctk_geom* g, int v, const double* b, double lam, const ctk_solver_opts* o, double* x, ctk_solve_log* l) { return ctk_lsmr_f64(g, v, b, lam, o, x, l); }
    static int hybrid(ctk_geom* g, int v, const double* b, const ctk_hybrid_strategy* s, const ctk_solver_opts* o, double* x, ctk_solve_log* l) { return ctk_hybrid_lsqr_f64(g, v, b, s, o, x, l); }
    static int flsqr_tv(ctk_geom* g, int v, const double* b, const ctk_hybrid_strategy* s, const ctk_solver_opts* o, double* x, ctk_solve_log* l) { return ctk_flsqr_tv_f64(g, v, b, s, o, x, l); }
    static int tv(ctk_geom* g, int v, const double* b, double lam, int oi, int ii, const ctk_solver_opts* o, int w, double* x, ctk_solve_log* l) { return ctk_cgls_tv_f64(g, v, b, lam, oi, ii, o, w, x, l); }
};

/// A ctk::OperatorPair<T> backed by the B200 kernels, plus the native handle the
/// device-resident solvers below run on.
template <class T>
struct B200Pair : ctk::OperatorPair<T> {
    std::shared_ptr<Handle> native;
    int variant = CTK_BP_MATCHED;
};

/// Drop-in for ctk::projector_pair<T> (operators.hpp:91-115): same validation and
/// canonicalisation, same overwrite-the-output semantics (operators.hpp:102-113).
template <class T>
B200Pair<T> projector_pair(const ctk::ConeGeometry& geom,
                           ctk::BackprojectVariant variant = ctk::BackprojectVariant::matched) {
    geom.validate();
    ctk::ConeGeometry g = geom;
    for (double& a : g.angles) a = ctk::canonical_angle(a);
    auto h = std::make_shared<Handle>(g);
    const int v = variant == ctk::BackprojectVariant::matched ? CTK_BP_MATCHED : CTK_BP_VOXEL_DRIVEN;
    B200Pair<T> p;
    p.domain_size = g.vol.size();
    p.range_size = g.proj_shape().size();
    p.matched = (v == CTK_BP_MATCHED);
    p.domain_shape = g.vol;
    p.forward = [h](std::span<const T> x, std::span<T> y) { check(Ops<T>::ax(h->get(), x.data(), y.data())); };
    p.back = [h, v](std::span<const T> y, std::span<T> x) { check(Ops<T>::atb(h->get(), v, y.data(), x.data())); };
    p.native = h;
    p.variant = v;
    return p;
}

namespace detail {

template <class T>
struct Call {
    std::vector<double> impl, expl, err, lam;
    std::vector<int> outer, warn;
    std::vector<T> gt;
    ctk_solve_log log{};
    ctk_solver_opts o{};
    const ctk::SolverOptions<T>* opts;

    Call(const ctk::OperatorPair<T>& pair, const ctk::SolverOptions<T>& so, int cap, int outer_cap) : opts(&so) {
        // IterationMonitor's constructor check (solve_log.hpp:92-94): a ground truth of the
        // wrong length is a DimensionError before any work
        if (so.ground_truth) pair.check_domain(so.ground_truth->size());
        impl.resize(size_t(cap));
        expl.resize(size_t(cap));
        err.resize(size_t(cap));
        lam.resize(size_t(cap));
        outer.resize(size_t(outer_cap) + 1);
        warn.resize(size_t(cap) + 1);
        log.capacity = cap;
        log.implicit_residual = impl.data();
        log.explicit_residual = expl.data();
        log.relative_error = err.data();
        log.lambda = lam.data();
        log.outer_starts = outer.data();
        log.warning_iterations = warn.data();
        o.max_iters = so.max_iters;
        o.stop_on_explicit_residual_increase = so.stop_on_explicit_residual_increase;
        o.residual_tolerance = so.residual_tolerance;
        o.reorth = so.reorth;
        if (so.ground_truth) {
            gt = *so.ground_truth;
            o.ground_truth = gt.data();
        }
        if (so.iterate_observer) {
            o.iterate_observer = [](int k, const void* hx, size_t n, void* user) {
                static_cast<Call*>(user)->opts->iterate_observer(k, std::span<const T>(static_cast<const T*>(hx), n));
            };
            o.observer_user = this;
        }
    }

    ctk::SolveResult<T> result(std::vector<T> x, const ctk::OperatorPair<T>& pair, const char* solver) {
        ctk::SolveResult<T> r;
        r.x = std::move(x);
        r.shape = pair.domain_shape;
        r.iterations_run = log.iterations_run;
        r.stop_reason = ctk::StopReason(log.stop_reason);
        r.log.implicit_residual.assign(impl.begin(), impl.begin() + log.iterations);
        r.log.explicit_residual.assign(expl.begin(), expl.begin() + log.iterations);
        r.log.relative_error.assign(err.begin(), err.begin() + log.n_relative_error);
        r.log.lambda.assign(lam.begin(), lam.begin() + log.n_lambda);
        r.log.solver = solver;
        r.log.precision = sizeof(T) == sizeof(double) ? "double" : "single";
        r.log.matched = pair.matched;
        r.outer_starts.assign(outer.begin(), outer.begin() + log.n_outer_starts);
        r.stored_domain_basis = log.stored_domain_basis;
        r.stored_range_basis = log.stored_range_basis;
        for (int i = 0; i < log.n_warnings; ++i)
            r.warnings.push_back("tv preconditioner: inner CG not converged at iteration " + std::to_string(warn[size_t(i)]));
        return r;
    }
};

}  // namespace detail

// Device-resident drop-ins for the reference solvers; same signatures, same SolveResult.
template <class T>
ctk::SolveResult<T> cgls(const B200Pair<T>& pair, std::span<const T> b, const ctk::SolverOptions<T>& opts) {
    opts.validate();
    pair.check_range(b.size());
    detail::Call<T> c(pair, opts, opts.max_iters, 1);
    std::vector<T> x(pair.domain_size);
    check(Ops<T>::cgls(pair.native->get(), pair.variant, b.data(), &c.o, x.data(), &c.log));
    return c.result(std::move(x), pair, "cgls");
}
template <class T>
ctk::SolveResult<T> lsqr(const B200Pair<T>& pair, std::span<const T> b, const ctk::SolverOptions<T>& opts) {
    opts.validate();
    pair.check_range(b.size());
    detail::Call<T> c(pair, opts, opts.max_iters, 1);
    std::vector<T> x(pair.domain_size);
    check(Ops<T>::lsqr(pair.native->get(), pair.variant, b.data(), &c.o, x.data(), &c.log));
    return c.result(std::move(x), pair, "lsqr");
}
/// SIRT (solvers.hpp:236-287)
template <class T>
ctk::SolveResult<T> sirt(const B200Pair<T>& pair, std::span<const T> b, const ctk::SolverOptions<T>& opts) {
    opts.validate();
    pair.check_range(b.size());
    detail::Call<T> c(pair, opts, opts.max_iters, 1);
    std::vector<T> x(pair.domain_size);
    check(Ops<T>::sirt(pair.native->get(), pair.variant, b.data(), &c.o, x.data(), &c.log));
    return c.result(std::move(x), pair, "sirt");
}
/// AB-GMRES / BA-GMRES (gmres.hpp:101-113)
template <class T>
ctk::SolveResult<T> ab_gmres(const B200Pair<T>& pair, std::span<const T> b, const ctk::SolverOptions<T>& opts) {
    opts.validate();
    pair.check_range(b.size());
    detail::Call<T> c(pair, opts, opts.max_iters, 1);
    std::vector<T> x(pair.domain_size);
    check(Ops<T>::ab_gmres(pair.native->get(), pair.variant, b.data(), &c.o, x.data(), &c.log));
    return c.result(std::move(x), pair, "ab_gmres");
}
template <class T>
ctk::SolveResult<T> ba_gmres(const B200Pair<T>& pair, std::span<const T> b, const ctk::SolverOptions<T>& opts) {
    opts.validate();
    pair.check_range(b.size());
    detail::Call<T> c(pair, opts, opts.max_iters, 1);
    std::vector<T> x(pair.domain_size);
    check(Ops<T>::ba_gmres(pair.native->get(), pair.variant, b.data(), &c.o, x.data(), &c.log));
    return c.result(std::move(x), pair, "ba_gmres");
}
template <class T>
ctk::SolveResult<T> lsmr(const B200Pair<T>& pair, std::span<const T> b, double lambda,
                         const ctk::SolverOptions<T>& opts) {
    opts.validate();
    pair.check_range(b.size());
    if (lambda < 0.0) throw ctk::ParameterError("lsmr: lambda must be nonnegative");
    detail::Call<T> c(pair, opts, opts.max_iters, 1);
    std::vector<T> x(pair.domain_size);
    check(Ops<T>::lsmr(pair.native->get(), pair.variant, b.data(), lambda, &c.o, x.data(), &c.log));
    return c.result(std::move(x), pair, "lsmr");
}
/// Strategy: ctk::HybridStrategy (hybrid.hpp:15-33) or anything with kind/lambda/noise_level.
template <class T, class Strategy>
ctk::SolveResult<T> hybrid_lsqr(const B200Pair<T>& pair, std::span<const T> b, const Strategy& s,
                                const ctk::SolverOptions<T>& opts) {
    opts.validate();
    pair.check_range(b.size());
    detail::Call<T> c(pair, opts, opts.max_iters, 1);
    std::vector<T> x(pair.domain_size);
    const ctk_hybrid_strategy cs{int(s.kind), s.lambda, s.noise_level};
    check(Ops<T>::hybrid(pair.native->get(), pair.variant, b.data(), &cs, &c.o, x.data(), &c.log));
    return c.result(std::move(x), pair, "hybrid_lsqr");
}
/// flsqr_tv (tv.hpp:177-185); Strategy as for hybrid_lsqr (fixed or gcv)
template <class T, class Strategy>
ctk::SolveResult<T> flsqr_tv(const B200Pair<T>& pair, std::span<const T> b, const Strategy& s,
                             const ctk::SolverOptions<T>& opts) {
    opts.validate();
    pair.check_range(b.size());
    detail::Call<T> c(pair, opts, opts.max_iters, 1);
    std::vector<T> x(pair.domain_size);
    const ctk_hybrid_strategy cs{int(s.kind), s.lambda, s.noise_level};
    check(Ops<T>::flsqr_tv(pair.native->get(), pair.variant, b.data(), &cs, &c.o, x.data(), &c.log));
    return c.result(std::move(x), pair, "flsqr_tv");
}
template <class T>
ctk::SolveResult<T> cgls_tv(const B200Pair<T>& pair, std::span<const T> b, double lambda, int outer_iters,
                            int inner_iters, const ctk::SolverOptions<T>& opts, bool warm_start = false) {
    opts.validate();
    pair.check_range(b.size());
    detail::Call<T> c(pair, opts, std::max(1, outer_iters) * std::max(1, inner_iters), std::max(1, outer_iters));
    std::vector<T> x(pair.domain_size);
    check(Ops<T>::tv(pair.native->get(), pair.variant, b.data(), lambda, outer_iters, inner_iters, &c.o,
                     int(warm_start), x.data(), &c.log));
    return c.result(std::move(x), pair, "cgls_tv");
}

}  // namespace ctkb
