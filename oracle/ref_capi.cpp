// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference headers (/root/reference/proj/include),
// compiled by oracle/Makefile into oracle/_ref/libctkref.so with the reference's
// Release flags (-O3 -DNDEBUG -std=c++20 -fopenmp, no -march=native).  Used to pin
// the C restatement (oracle/ctk_oracle.c) and as the CPU baseline ("kind": "reference").
// No reference source is copied here; the reference is #included from where it lies.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <exception>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "ctkrylov/io.hpp"
#include "ctkrylov/noise.hpp"
#include "ctkrylov/operators.hpp"
#include "ctkrylov/phantom.hpp"
#include "ctkrylov/solvers.hpp"
#ifdef CTK_REF_WITH_EIGEN
#include "ctkrylov/gmres.hpp"
#include "ctkrylov/hybrid.hpp"
#include "ctkrylov/regparam.hpp"
#include "ctkrylov/tv.hpp"
#endif

extern "C" {

struct ref_geom {
    int mode;
    double dso, dod, du;
    int nu, nv;
    int nx, ny, nz;
    double h;
    int na;
    const double* angles;
};

struct ref_log {
    double* implicit_residual;  // capacity = max_iters each
    double* explicit_residual;
    double* relative_error;
    double* lambda;
    int iterations;
    int n_relerr;
    int n_lambda;
    int iterations_run;
    int stop_reason;
    int error_iteration;
    int* outer_starts;
    int n_outer_starts;
    int stored_domain_basis;
    int stored_range_basis;
    int* warning_iterations;  // SolveResult::warnings: the trailing iteration number of each
    int n_warnings;
};

}  // extern "C"

namespace {

ctk::ConeGeometry to_geom(const ref_geom* d) {
    ctk::ConeGeometry g;
    g.mode = d->mode == 0 ? ctk::BeamMode::parallel2d
                          : (d->mode == 1 ? ctk::BeamMode::parallel3d : ctk::BeamMode::cone3d);
    g.source_to_origin = d->dso;
    g.origin_to_detector = d->dod;
    g.detector_pixel_size = d->du;
    g.nu = d->nu;
    g.nv = d->nv;
    g.vol = {d->nx, d->ny, d->nz, d->h};
    g.angles.assign(d->angles, d->angles + d->na);
    return g;
}

int g_err_iter = 0;
std::string g_err_msg;

template <class F>
int guarded(F&& f) {
    g_err_msg.clear();
    try {
        f();
        return 0;
    } catch (const ctk::DimensionError& e) {
        g_err_msg = e.what();
        return 1;
    } catch (const ctk::GeometryError& e) {
        g_err_msg = e.what();
        return 2;
    } catch (const ctk::ParameterError& e) {
        g_err_msg = e.what();
        return 3;
    } catch (const ctk::DegenerateInputError& e) {
        g_err_msg = e.what();
        return 4;
    } catch (const ctk::NumericalError& e) {
        g_err_iter = e.iteration;
        g_err_msg = e.what();
        return 5;
    } catch (...) {
        return 9;
    }
}

template <typename T>
int forward_impl(const ref_geom* d, const T* x, T* y) {
    return guarded([&] {
        auto g = to_geom(d);
        auto pair = ctk::projector_pair<T>(g, ctk::BackprojectVariant::matched);
        std::vector<T> out = pair.apply_forward(std::span<const T>(x, pair.domain_size));
        std::memcpy(y, out.data(), out.size() * sizeof(T));
    });
}

template <typename T>
int back_impl(const ref_geom* d, int variant, const T* y, T* x) {
    return guarded([&] {
        auto g = to_geom(d);
        auto v = variant == 0 ? ctk::BackprojectVariant::matched : ctk::BackprojectVariant::voxel_driven;
        auto pair = ctk::projector_pair<T>(g, v);
        std::vector<T> out = pair.apply_back(std::span<const T>(y, pair.range_size));
        std::memcpy(x, out.data(), out.size() * sizeof(T));
    });
}

template <typename T>
void fill_log(const ctk::SolveResult<T>& r, ref_log* log) {
    const auto& L = r.log;
    log->iterations = int(L.explicit_residual.size());
    for (std::size_t i = 0; i < L.explicit_residual.size(); ++i) {
        log->implicit_residual[i] = L.implicit_residual[i];
        log->explicit_residual[i] = L.explicit_residual[i];
    }
    log->n_relerr = int(L.relative_error.size());
    for (std::size_t i = 0; i < L.relative_error.size(); ++i) log->relative_error[i] = L.relative_error[i];
    log->n_lambda = int(L.lambda.size());
    for (std::size_t i = 0; i < L.lambda.size(); ++i) log->lambda[i] = L.lambda[i];
    log->iterations_run = r.iterations_run;
    log->stop_reason = int(r.stop_reason);
    log->n_outer_starts = int(r.outer_starts.size());
    if (log->outer_starts)
        for (std::size_t i = 0; i < r.outer_starts.size(); ++i) log->outer_starts[i] = r.outer_starts[i];
    log->stored_domain_basis = r.stored_domain_basis;
    log->stored_range_basis = r.stored_range_basis;
    log->n_warnings = int(r.warnings.size());
    if (log->warning_iterations)
        for (std::size_t i = 0; i < r.warnings.size(); ++i) {
            const std::string& w = r.warnings[i];
            log->warning_iterations[i] = std::atoi(w.c_str() + w.find_last_of(' ') + 1);
        }
}

// solver: 0 cgls, 1 lsqr, 2 lsmr, 3 sirt, 4 hybrid_lsqr, 5 cgls_tv, 6 ab_gmres, 7 ba_gmres, 8 flsqr_tv
template <typename T>
int solve_impl(const ref_geom* d, int variant, int solver, double lambda, int strategy,
               double noise_level, int outer, int inner, int warm, const T* b, int max_iters,
               double tol, int stop_inc, int reorth, const T* gt, T* x_out, ref_log* log) {
    g_err_iter = 0;
    int rc = guarded([&] {
        auto g = to_geom(d);
        auto v = variant == 0 ? ctk::BackprojectVariant::matched : ctk::BackprojectVariant::voxel_driven;
        auto pair = ctk::projector_pair<T>(g, v);
        ctk::SolverOptions<T> opts;
        opts.max_iters = max_iters;
        opts.residual_tolerance = tol;
        opts.stop_on_explicit_residual_increase = stop_inc != 0;
        opts.reorth = reorth != 0;
        if (gt) opts.ground_truth = std::vector<T>(gt, gt + pair.domain_size);
        std::span<const T> bs(b, pair.range_size);
        ctk::SolveResult<T> r;
        switch (solver) {
            case 0: r = ctk::cgls(pair, bs, opts); break;
            case 1: r = ctk::lsqr(pair, bs, opts); break;
            case 2: r = ctk::lsmr(pair, bs, lambda, opts); break;
            case 3: r = ctk::sirt(pair, bs, opts); break;
#ifdef CTK_REF_WITH_EIGEN
            case 4: {
                ctk::HybridStrategy s = strategy == 0 ? ctk::HybridStrategy::fixed(lambda)
                                      : strategy == 1 ? ctk::HybridStrategy::dp(noise_level)
                                                      : ctk::HybridStrategy::gcv();
                r = ctk::hybrid_lsqr(pair, bs, s, opts);
                break;
            }
            case 5: r = ctk::cgls_tv(pair, bs, lambda, outer, inner, opts, warm != 0); break;
            case 6: r = ctk::ab_gmres(pair, bs, opts); break;
            case 7: r = ctk::ba_gmres(pair, bs, opts); break;
            case 8: {
                ctk::HybridStrategy s = strategy == 0 ? ctk::HybridStrategy::fixed(lambda) : ctk::HybridStrategy::gcv();
                r = ctk::flsqr_tv(pair, bs, s, opts);
                break;
            }
#endif
            default: throw ctk::ParameterError("solver not available in this build");
        }
        std::memcpy(x_out, r.x.data(), r.x.size() * sizeof(T));
        fill_log(r, log);
    });
    log->error_iteration = g_err_iter;
    (void)strategy;
    (void)noise_level;
    (void)outer;
    (void)inner;
    (void)warm;
    return rc;
}

}  // namespace

extern "C" {

int ref_has_eigen() {
#ifdef CTK_REF_WITH_EIGEN
    return 1;
#else
    return 0;
#endif
}

void ref_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int ref_max_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

int ref_forward_f64(const ref_geom* d, const double* x, double* y) { return forward_impl(d, x, y); }
int ref_forward_f32(const ref_geom* d, const float* x, float* y) { return forward_impl(d, x, y); }
int ref_back_f64(const ref_geom* d, int variant, const double* y, double* x) { return back_impl(d, variant, y, x); }
int ref_back_f32(const ref_geom* d, int variant, const float* y, float* x) { return back_impl(d, variant, y, x); }

int ref_solve_f64(const ref_geom* d, int variant, int solver, double lambda, int strategy,
                  double noise_level, int outer, int inner, int warm, const double* b,
                  int max_iters, double tol, int stop_inc, int reorth, const double* gt,
                  double* x, ref_log* log) {
    return solve_impl(d, variant, solver, lambda, strategy, noise_level, outer, inner, warm, b,
                      max_iters, tol, stop_inc, reorth, gt, x, log);
}
int ref_solve_f32(const ref_geom* d, int variant, int solver, double lambda, int strategy,
                  double noise_level, int outer, int inner, int warm, const float* b,
                  int max_iters, double tol, int stop_inc, int reorth, const float* gt,
                  float* x, ref_log* log) {
    return solve_impl(d, variant, solver, lambda, strategy, noise_level, outer, inner, warm, b,
                      max_iters, tol, stop_inc, reorth, gt, x, log);
}

// kind: 0 shepp_logan_3d, 1 shepp_logan_2d, 2 piecewise_blocks
int ref_phantom_f64(int kind, int n, double* out) {
    return guarded([&] {
        auto k = kind == 0 ? ctk::PhantomKind::shepp_logan_3d
               : kind == 1 ? ctk::PhantomKind::shepp_logan_2d
                           : ctk::PhantomKind::piecewise_blocks;
        auto v = ctk::make_phantom<double>(k, n);
        std::memcpy(out, v.data.data(), v.data.size() * sizeof(double));
    });
}
int ref_phantom_f32(int kind, int n, float* out) {
    return guarded([&] {
        auto k = kind == 0 ? ctk::PhantomKind::shepp_logan_3d
               : kind == 1 ? ctk::PhantomKind::shepp_logan_2d
                           : ctk::PhantomKind::piecewise_blocks;
        auto v = ctk::make_phantom<float>(k, n);
        std::memcpy(out, v.data.data(), v.data.size() * sizeof(float));
    });
}

int ref_add_noise_f64(const ref_geom* d, const double* clean, double i0, double sigma,
                      std::uint64_t seed, double* out) {
    return guarded([&] {
        ctk::ProjectionSet<double> p(std::vector<double>(d->angles, d->angles + d->na), d->nu, d->nv);
        std::memcpy(p.data.data(), clean, p.data.size() * sizeof(double));
        auto r = ctk::add_noise(p, ctk::NoiseModel{i0, sigma, seed});
        std::memcpy(out, r.data.data(), r.data.size() * sizeof(double));
    });
}

int ref_gradient_f64(int nx, int ny, int nz, const double* v, double* dx, double* dy, double* dz) {
    return guarded([&] {
        ctk::Volume<double> vol(nx, ny, nz, 1.0);
        std::memcpy(vol.data.data(), v, vol.size() * sizeof(double));
        auto g = ctk::gradient(vol);
        std::memcpy(dx, g.dx.data(), vol.size() * sizeof(double));
        std::memcpy(dy, g.dy.data(), vol.size() * sizeof(double));
        std::memcpy(dz, g.dz.data(), vol.size() * sizeof(double));
    });
}

int ref_gradient_adjoint_f64(int nx, int ny, int nz, const double* dx, const double* dy,
                             const double* dz, double* out) {
    return guarded([&] {
        ctk::GradientField<double> g(ctk::VolumeShape{nx, ny, nz, 1.0});
        const std::size_t n = g.dx.size();
        std::memcpy(g.dx.data(), dx, n * sizeof(double));
        std::memcpy(g.dy.data(), dy, n * sizeof(double));
        std::memcpy(g.dz.data(), dz, n * sizeof(double));
        auto v = ctk::gradient_adjoint(g);
        std::memcpy(out, v.data.data(), n * sizeof(double));
    });
}

#ifdef CTK_REF_WITH_EIGEN
int ref_tv_weights_f64(int nx, int ny, int nz, const double* x, double* w) {
    return guarded([&] {
        ctk::Volume<double> vol(nx, ny, nz, 1.0);
        std::memcpy(vol.data.data(), x, vol.size() * sizeof(double));
        auto ww = ctk::tv_weights(vol);
        std::memcpy(w, ww.data(), ww.size() * sizeof(double));
    });
}

// Projected-problem parameter choice on an explicit (k+1) x k matrix (row-major).
double ref_gcv_lambda(const double* H, int k, double beta1) {
    Eigen::MatrixXd m = Eigen::MatrixXd::Zero(k + 1, k);
    for (int i = 0; i < k + 1; ++i)
        for (int j = 0; j < k; ++j) m(i, j) = H[i * k + j];
    ctk::ProjectedProblem p{m, beta1, k};
    return ctk::gcv_lambda(p);
}
double ref_dp_lambda(const double* H, int k, double beta1, double nl) {
    Eigen::MatrixXd m = Eigen::MatrixXd::Zero(k + 1, k);
    for (int i = 0; i < k + 1; ++i)
        for (int j = 0; j < k; ++j) m(i, j) = H[i * k + j];
    ctk::ProjectedProblem p{m, beta1, k};
    return ctk::dp_lambda(p, nl);
}
#endif

}  // extern "C"

// ---- raw f32 + .hdr I/O and 16-bit PGM (src/io.cpp, compiled from where it lies) ----------
extern "C" {
int ref_save_volume(const char* path, int nx, int ny, int nz, double spacing, const float* data) {
    return guarded([&] {
        ctk::Volume<float> v(nx, ny, nz, spacing);
        std::memcpy(v.data.data(), data, v.data.size() * sizeof(float));
        ctk::save_volume(path, v);
    });
}
// shape[4] = nx ny nz + spacing in *spacing; data may be NULL (header only)
int ref_load_volume(const char* path, int* shape, double* spacing, float* data, size_t cap) {
    return guarded([&] {
        const auto v = ctk::load_volume(path);
        shape[0] = v.nx;
        shape[1] = v.ny;
        shape[2] = v.nz;
        *spacing = v.spacing;
        if (data && cap >= v.data.size()) std::memcpy(data, v.data.data(), v.data.size() * sizeof(float));
    });
}
int ref_save_projections(const char* path, int na, int nu, int nv, const double* angles, const float* data) {
    return guarded([&] {
        ctk::ProjectionSet<float> p(std::vector<double>(angles, angles + na), nu, nv);
        std::memcpy(p.data.data(), data, p.data.size() * sizeof(float));
        ctk::save_projections(path, p);
    });
}
int ref_load_projections(const char* path, int* dims, double* angles, size_t angle_cap, float* data, size_t cap) {
    return guarded([&] {
        const auto p = ctk::load_projections(path);
        dims[0] = p.n_angles;
        dims[1] = p.nu;
        dims[2] = p.nv;
        if (angles && angle_cap >= p.angles.size()) std::memcpy(angles, p.angles.data(), p.angles.size() * sizeof(double));
        if (data && cap >= p.data.size()) std::memcpy(data, p.data.data(), p.data.size() * sizeof(float));
    });
}
int ref_write_pgm16(const char* path, int w, int h, const float* values, double wmin, double wmax) {
    return guarded([&] { ctk::write_pgm16(path, w, h, values, wmin, wmax); });
}
}  // extern "C"

// ---- pipeline, config, metrics (src/config.cpp, src/pipeline.cpp compiled from where
//      they lie; include/ctkrylov/{config,pipeline,metrics,noise}.hpp) ----------------------
#ifdef CTK_REF_WITH_EIGEN
#include <fstream>
#include <sstream>

#include "ctkrylov/config.hpp"
#include "ctkrylov/metrics.hpp"
#include "ctkrylov/pipeline.hpp"

extern "C" {
int ref_last_error_message(char* buf, size_t cap) {
    if (cap) {
        std::strncpy(buf, g_err_msg.c_str(), cap - 1);
        buf[cap - 1] = 0;
    }
    return int(g_err_msg.size());
}

int ref_add_noise_f32(const ref_geom* d, const float* clean, double i0, double sigma, std::uint64_t seed,
                      float* out) {
    return guarded([&] {
        ctk::ProjectionSet<float> p(std::vector<double>(d->angles, d->angles + d->na), d->nu, d->nv);
        std::memcpy(p.data.data(), clean, p.data.size() * sizeof(float));
        auto r = ctk::add_noise(p, ctk::NoiseModel{i0, sigma, seed});
        std::memcpy(out, r.data.data(), r.data.size() * sizeof(float));
    });
}

// cmd: 0 simulate, 1 reconstruct, 2 compare; cfg_text is a key = value config
int ref_run_pipeline(int cmd, const char* cfg_text) {
    return guarded([&] {
        std::istringstream in(cfg_text);
        ctk::RunConfig cfg = ctk::parse_config(in);
        if (cmd == 0) ctk::run_simulate(cfg);
        else if (cmd == 1) ctk::run_reconstruct(cfg);
        else ctk::run_compare(cfg);
    });
}

// parse_config(cfg_text) then write_config to out_path (resolve != 0: resolve_geometry first)
int ref_config_write(const char* cfg_text, int resolve, const char* out_path) {
    return guarded([&] {
        std::istringstream in(cfg_text);
        ctk::RunConfig cfg = ctk::parse_config(in);
        if (resolve) ctk::resolve_geometry(cfg);
        std::ofstream f(out_path);
        ctk::write_config(f, cfg);
    });
}

// resolve_geometry(cfg): geometry out (angles into a caller buffer of >= n_angles)
int ref_resolve_geometry(const char* cfg_text, ref_geom* out, double* angles) {
    return guarded([&] {
        std::istringstream in(cfg_text);
        ctk::RunConfig cfg = ctk::parse_config(in);
        const ctk::ConeGeometry g = ctk::resolve_geometry(cfg);
        out->mode = int(g.mode);
        out->dso = g.source_to_origin;
        out->dod = g.origin_to_detector;
        out->du = g.detector_pixel_size;
        out->nu = g.nu;
        out->nv = g.nv;
        out->nx = g.vol.nx;
        out->ny = g.vol.ny;
        out->nz = g.vol.nz;
        out->h = g.vol.spacing;
        out->na = int(g.angles.size());
        std::memcpy(angles, g.angles.data(), g.angles.size() * sizeof(double));
    });
}

// write_csv of a log given its four columns (metrics.hpp:80-91)
int ref_write_csv(const char* path, const double* impl, int n_impl, const double* expl, int n_expl,
                  const double* err, int n_err, const double* lam, int n_lam) {
    return guarded([&] {
        ctk::ConvergenceLog log;
        log.implicit_residual.assign(impl, impl + n_impl);
        log.explicit_residual.assign(expl, expl + n_expl);
        log.relative_error.assign(err, err + n_err);
        log.lambda.assign(lam, lam + n_lam);
        std::ofstream f(path);
        ctk::write_csv(f, log);
    });
}

// detect_semiconvergence / residual_divergence (metrics.hpp:40-75)
int ref_semiconvergence(const double* err, int n, int* min_index, double* rebound) {
    return guarded([&] {
        ctk::ConvergenceLog log;
        log.relative_error.assign(err, err + n);
        const auto s = ctk::detect_semiconvergence(log);
        *min_index = s.min_index;
        *rebound = s.rebound_ratio;
    });
}
int ref_residual_divergence(const double* impl, int n_impl, const double* expl, int n_expl, double* out) {
    return guarded([&] {
        ctk::ConvergenceLog log;
        log.implicit_residual.assign(impl, impl + n_impl);
        log.explicit_residual.assign(expl, expl + n_expl);
        *out = ctk::residual_divergence(log);
    });
}
}  // extern "C"
#endif
