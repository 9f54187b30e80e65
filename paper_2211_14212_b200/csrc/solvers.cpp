// Device-resident Krylov solvers.  Control flow, stopping rules, breakdown tests and log
// semantics follow the reference line by line; vectors live in HBM and every vector
// operation is one of the fused kernels of blas1.cu / kernels_f32.cu / kernels_f64.cu.
// Scalar recurrences run on the host in fp64 (the reference runs them in T; for T=double
// they are the same operations).
//   IterationMonitor   solve_log.hpp:86-161     cgls         solvers.hpp:13-60
//   lsqr               solvers.hpp:62-126       lsmr         solvers.hpp:128-231
//   hybrid_lsqr        hybrid.hpp:76-116 (gk_init/gk_expand krylov.hpp:50-92, cgs2 :21-31)
//   cgls_tv            tv.hpp:45-110 (stack_weighted_gradient operators.hpp:141-186)
// With a communicator attached the vectors of one space are sharded and the other is
// replicated:
//   angle sharding  range vectors are this rank's angle block; range reductions are summed
//                   over ranks in rank order and every A^T b partial volume is sum-reduced,
//                   so all ranks hold identical domain vectors;
//   z-slab          domain vectors are this rank's slab of z-slices; domain reductions are
//                   summed in rank order and every A x partial projection set is
//                   sum-reduced (by linearity A x = sum_r A x_r), so all ranks hold
//                   identical range vectors; the TV stencils exchange one-slice halos;
//   z-slab + band   (ctk_geom_shard_range) range vectors hold the rank's detector-row window
//                   too: A x partials go to the rows' owners, A^T b fetches its halo rows
//                   (bands.cpp) and range reductions are summed over ranks as well.
#include <algorithm>
#include <cmath>
#include <string>
#include <utility>
#include <vector>

#include "ctk_internal.h"
#include "regparam.h"

namespace ctkb {
namespace {

template <class T>
constexpr double breakdown_factor() {  // krylov.hpp:14-17
    return sizeof(T) == sizeof(double) ? 1e-14 : 1e-7;
}
constexpr double kIncreaseSlack = 1e-12;  // solve_log.hpp:80

// the handle whose workspace pool the current solve draws from (solve_device sets it)
thread_local Geometry* t_pool = nullptr;
DevBuf& pooled() {
    if (!t_pool) fail(CTK_E_PARAMETER, "solver workspace requested outside a solve");
    return t_pool->ws_take();
}

template <class T>
struct Vec {
    DevBuf* buf = nullptr;
    size_t n = 0;
    T* p = nullptr;
    void alloc(size_t nn) {
        n = nn;
        if (!buf) buf = &pooled();
        buf->ensure(sizeof(T) * std::max<size_t>(nn, 1));
        p = buf->as<T>();
    }
};

// Device operator + reductions for one solve.
template <class T>
struct Dev {
    Geometry& g;
    int variant;
    cudaStream_t s;
    RedWork w;
    Vec<T> tmp_range;  // explicit residual staging (f64 path)

    Dev(Geometry& g_, int v) : g(g_), variant(v), s(g_.stream), w(red_work(&g_)) {}

    bool slab_mode() const { return g.comm && g.slab; }
    // are vectors of this space split across ranks (their reductions summed)?  With the
    // band-sharded range (bands.cpp) both spaces are: range vectors hold this rank's row
    // window with the rows it does not own at zero
    bool sharded(bool range) const { return g.comm && (g.slab ? (!range || g.band) : range); }
    // The solver's next forward application, announced before the monitor records an
    // iterate: the explicit residual's A x and that A v then run as one two-volume march
    // (ax2_f32), and the next ax(v, y) finds y already written.  Only the solvers that leave
    // v and y untouched between record() and that call announce it (lsqr, lsmr, hybrid_lsqr).
    const T* next_in = nullptr;
    T* next_out = nullptr;
    bool next_ready = false;
    // can the monitor's A x run paired with a following forward application?
    bool can_pair() const { return sizeof(T) == 4 && ax2_f32_supported(g); }
    void announce_ax(const T* x, T* y) {
        next_in = x;
        next_out = y;
        next_ready = false;
    }
    void ax(const T* x, T* y) {
        const bool ready = next_ready && x == next_in && y == next_out;
        next_in = nullptr;
        next_out = nullptr;
        next_ready = false;
        if (ready) return;
        op_ax<T>(g, x, y, s);
        if (slab_mode()) {
            if (g.band) band_reduce<T>(g, y, s);  // partials to the rows' owners, rank order
            else comm_allreduce(g.comm, y, g.range(), sizeof(T) == 8 ? 1 : 0, s);
        }
    }
    void atb(const T* y, T* x) {
        next_ready = false;
        op_atb<T>(g, variant, g.band ? band_halo<T>(g, y, s) : y, x, s);
        if (g.comm && !g.slab) comm_allreduce(g.comm, x, g.domain(), sizeof(T) == 8 ? 1 : 0, s);
    }
    double fetch(int slot) {
        CTK_CUDA(cudaMemcpyAsync(g.pinned + slot, w.results + slot, sizeof(double), cudaMemcpyDeviceToHost, s));
        CTK_CUDA(cudaStreamSynchronize(s));
        return g.pinned[slot];
    }
    double part_sum(double v, bool range) { return sharded(range) ? comm_sum_scalar(g.comm, v) : v; }
    double domain_max(double v) { return sharded(false) ? comm_max_scalar(g.comm, v) : v; }

    // ---- one-slice halos of z-slab sharding (gradient.hpp:19-21 and its transpose) ----
    // Every rank's chosen slice is gathered by a sum-allreduce of a zeroed [nranks][nx*ny]
    // buffer in which each rank fills only its own row: one nonzero term per entry, exact.
    DevBuf* halo = nullptr;
    bool last_slab() const { return g.comm->cb.rank == g.comm->cb.nranks - 1; }
    const T* gather_slices(const T* slice) {
        const size_t S = size_t(g.nx) * g.ny, R = size_t(g.comm->cb.nranks);
        if (!halo) halo = &pooled();
        halo->ensure(sizeof(T) * S * R);
        fill<T>(S * R, T(0), halo->as<T>(), s);
        CTK_CUDA(cudaMemcpyAsync(halo->as<T>() + size_t(g.comm->cb.rank) * S, slice, sizeof(T) * S,
                                 cudaMemcpyDeviceToDevice, s));
        comm_allreduce(g.comm, halo->p, S * R, sizeof(T) == 8 ? 1 : 0, s);
        return halo->as<T>();
    }
    // point-to-point halo when the transport has it (NCCL, or an exchange callback): send
    // `mine` to rank `to`, receive rank `from`'s slice into the halo buffer (-1: none)
    bool p2p() const { return g.comm->nccl_comm || g.comm->cb.exchange; }
    const T* swap_slice(const T* mine, int to, int from) {
        const size_t S = size_t(g.nx) * g.ny;
        if (!halo) halo = &pooled();
        halo->ensure(sizeof(T) * S);
        std::vector<ctk_p2p_op> ops;
        if (to >= 0) ops.push_back({to, 1, const_cast<T*>(mine), S});
        if (from >= 0) ops.push_back({from, 0, halo->p, S});
        comm_exchange(g.comm, ops, sizeof(T) == 8 ? 1 : 0, s);
        return from >= 0 ? halo->as<T>() : nullptr;
    }
    // the next rank's first slice of x (null when unsharded or on the last slab)
    const T* slice_above(const T* x) {
        if (!slab_mode()) return nullptr;
        const int r = g.comm->cb.rank;
        if (p2p()) return swap_slice(x, r > 0 ? r - 1 : -1, last_slab() ? -1 : r + 1);
        const T* all = gather_slices(x);
        return last_slab() ? nullptr : all + size_t(g.comm->cb.rank + 1) * size_t(g.nx) * g.ny;
    }
    // the previous rank's last slice of lam * w .* gz (null when unsharded or on the first slab)
    Vec<T> wtop;
    const T* weighted_slice_below(const T* gz, const T* wts, double lam) {
        if (!slab_mode()) return nullptr;
        const size_t S = size_t(g.nx) * g.ny, top = size_t(g.nz_local() - 1) * S;
        if (!wtop.p) wtop.alloc(S);
        if (wts) {
            scale_copy<T>(S, lam, wts + top, wtop.p, s);  // sc = lam * w   (operators.hpp:176-181)
            mul<T>(S, wtop.p, gz + top, wtop.p, s);
        } else {
            CTK_CUDA(cudaMemcpyAsync(wtop.p, gz + top, sizeof(T) * S, cudaMemcpyDeviceToDevice, s));
        }
        const int r = g.comm->cb.rank;
        if (p2p()) return swap_slice(wtop.p, last_slab() ? -1 : r + 1, r > 0 ? r - 1 : -1);
        const T* all = gather_slices(wtop.p);
        return g.comm->cb.rank == 0 ? nullptr : all + size_t(g.comm->cb.rank - 1) * S;
    }

    double nrm2sq(const T* x, size_t n, bool range) {
        reduce_dot<T>(n, x, x, w.results, w, s);
        const double v = fetch(0);
        return part_sum(v, range);
    }
    double diff_nrm2sq(const T* a, const T* b, size_t n, bool range) {
        reduce_diff_nrm2sq<T>(n, a, b, w.results, w, s);
        const double v = fetch(0);
        return part_sum(v, range);
    }
    // y += alpha x, returns ||y||^2
    double axpy_n2(double alpha, const T* x, T* y, size_t n, bool range) {
        axpy_nrm2sq<T>(n, alpha, x, y, w.results, w, s);
        const double v = fetch(0);
        return part_sum(v, range);
    }
    // ||A x - b||^2 over all ranks (solve_log.hpp:111-115), never storing A x in T=float
    double resid2(const T* x, const T* b) {
        if constexpr (sizeof(T) == 4) {
            if (next_in && !next_ready && ax2_f32_supported(g)) {
                if (!tmp_range.p) tmp_range.alloc(g.range());
                ax2_f32(g, reinterpret_cast<const float*>(next_in), reinterpret_cast<float*>(next_out), x,
                        reinterpret_cast<float*>(tmp_range.p), s);
                next_ready = true;
                return diff_nrm2sq(tmp_range.p, b, g.range(), true);
            }
            if (g.projector == CTK_PROJ_JOSEPH && !slab_mode()) {
                ax_residual_f32(g, x, b, w.results, s);
                return part_sum(fetch(0), true);
            }
        }
        {
            if (!tmp_range.p) tmp_range.alloc(g.range());
            ax(x, tmp_range.p);
            return diff_nrm2sq(tmp_range.p, b, g.range(), true);
        }
    }
};

template <class T>
struct Monitor {
    Dev<T>& d;
    const T* b;
    const ctk_solver_opts& o;
    ctk_solve_log* log;
    double bnorm = 0, gt_norm = 0, prev = 0;
    bool have_prev = false;
    int reason = CTK_STOP_MAX_ITERS;
    Vec<T> gt;
    std::vector<T> host_x;

    Monitor(Dev<T>& dev, const T* b_, const ctk_solver_opts& opts, ctk_solve_log* lg, const std::string& name)
        : d(dev), b(b_), o(opts), log(lg) {
        bnorm = std::sqrt(d.nrm2sq(b, d.g.range(), true));
        if (!(bnorm > 0.0)) fail(CTK_E_DEGENERATE, name + ": zero right-hand side");
        if (o.ground_truth) {
            gt.alloc(d.g.domain());
            CTK_CUDA(cudaMemcpyAsync(gt.p, o.ground_truth, sizeof(T) * d.g.domain(), cudaMemcpyHostToDevice, d.s));
            gt_norm = std::sqrt(d.nrm2sq(gt.p, d.g.domain(), false));
            if (!(gt_norm > 0.0)) fail(CTK_E_DEGENERATE, "ground truth has zero norm");
        }
        log->iterations = log->n_relative_error = log->n_lambda = log->n_warnings = 0;
    }

    // IterationMonitor::record; returns true when the solver should stop.  expl_override:
    // the relative explicit residual when the caller already formed it from a genuine
    // forward application of this iterate (solve_log.hpp:102-115; SIRT), else computed here.
    bool record(int k, const T* x, double implicit, bool has_lambda = false, double lambda = 0.0,
                const double* expl_override = nullptr) {
        const double expl = expl_override ? *expl_override : std::sqrt(d.resid2(x, b)) / bnorm;
        if (!std::isfinite(expl) || !std::isfinite(implicit))
            fail(CTK_E_NUMERICAL, "non-finite residual at iteration " + std::to_string(k), k);
        if (log->iterations >= log->capacity) fail(CTK_E_PARAMETER, "solve log capacity exceeded");
        log->implicit_residual[log->iterations] = implicit;
        log->explicit_residual[log->iterations] = expl;
        log->iterations++;
        if (has_lambda && log->lambda) log->lambda[log->n_lambda++] = lambda;
        if (o.ground_truth && log->relative_error)
            log->relative_error[log->n_relative_error++] =
                std::sqrt(d.diff_nrm2sq(x, gt.p, d.g.domain(), false)) / gt_norm;
        if (o.iterate_observer) {
            host_x.resize(d.g.domain());
            CTK_CUDA(cudaMemcpyAsync(host_x.data(), x, sizeof(T) * host_x.size(), cudaMemcpyDeviceToHost, d.s));
            CTK_CUDA(cudaStreamSynchronize(d.s));
            o.iterate_observer(k, host_x.data(), host_x.size(), o.observer_user);
        }
        if (expl <= o.residual_tolerance) {
            reason = CTK_STOP_TOLERANCE;
            return true;
        }
        if (o.stop_on_explicit_residual_increase && have_prev && expl > prev * (1.0 + kIncreaseSlack)) {
            reason = CTK_STOP_RESIDUAL_INCREASE;
            return true;
        }
        prev = expl;
        have_prev = true;
        return false;
    }
    void finish(int iterations) {
        log->iterations_run = iterations;
        log->stop_reason = reason;
    }
};

void validate_opts(const ctk_solver_opts* o, const ctk_solve_log* log, int need) {
    if (!o || !log) fail(CTK_E_PARAMETER, "null options or log");
    if (o->max_iters < 1) fail(CTK_E_PARAMETER, "max_iters must be >= 1");
    if (o->residual_tolerance < 0.0) fail(CTK_E_PARAMETER, "residual tolerance must be >= 0");
    if (!log->implicit_residual || !log->explicit_residual || log->capacity < need)
        fail(CTK_E_PARAMETER, "solve log needs capacity >= max iterations");
}

// ---------------------------------------------------------------------------------------
template <class T>
void cgls(Dev<T>& d, const T* b, const ctk_solver_opts& o, T* x, ctk_solve_log* log) {
    Geometry& g = d.g;
    const size_t nd = g.domain(), nr = g.range();
    Monitor<T> mon(d, b, o, log, "cgls");
    const double bnorm = mon.bnorm;
    Vec<T> r, s, p, q;
    r.alloc(nr); s.alloc(nd); p.alloc(nd); q.alloc(nr);
    fill<T>(nd, T(0), x, d.s);
    CTK_CUDA(cudaMemcpyAsync(r.p, b, sizeof(T) * nr, cudaMemcpyDeviceToDevice, d.s));
    d.atb(r.p, s.p);
    CTK_CUDA(cudaMemcpyAsync(p.p, s.p, sizeof(T) * nd, cudaMemcpyDeviceToDevice, d.s));
    double gamma = d.nrm2sq(s.p, nd, false);
    int k = 0;
    while (k < o.max_iters) {
        ++k;
        if (!(gamma > 0.0)) {
            mon.reason = CTK_STOP_BREAKDOWN;
            --k;
            break;
        }
        d.ax(p.p, q.p);
        const double delta = d.nrm2sq(q.p, nr, true);
        if (!std::isfinite(delta)) fail(CTK_E_NUMERICAL, "cgls: non-finite curvature at iteration " + std::to_string(k), k);
        if (!(delta > 0.0)) {
            mon.reason = CTK_STOP_BREAKDOWN;
            --k;
            break;
        }
        const double alpha = gamma / delta;
        axpy<T>(nd, alpha, p.p, x, d.s);
        const double rr = d.axpy_n2(-alpha, q.p, r.p, nr, true);
        auto advance = [&] {  // s = A^T r, p = s + beta p
            d.atb(r.p, s.p);
            const double gnew = d.nrm2sq(s.p, nd, false);
            const double beta = gnew / gamma;
            gamma = gnew;
            xpby<T>(nd, s.p, beta, p.p, d.s);
        };
        // With the two-volume march the recurrence advances before the monitor records x_k,
        // so its A x pairs with the next A p (the same values; on a stop the advance is unused)
        const bool ahead = k < o.max_iters && d.can_pair();
        if (ahead) {
            advance();
            d.announce_ax(p.p, q.p);
        }
        if (mon.record(k, x, std::sqrt(rr) / bnorm)) break;
        if (!ahead) advance();
    }
    mon.finish(k);
}

template <class T>
void lsqr(Dev<T>& d, const T* b, const ctk_solver_opts& o, T* x, ctk_solve_log* log) {
    Geometry& g = d.g;
    const size_t nd = g.domain(), nr = g.range();
    Monitor<T> mon(d, b, o, log, "lsqr");
    const double beta1 = mon.bnorm;
    const double tol = breakdown_factor<T>() * beta1;
    Vec<T> u, un, v, vn, w;
    u.alloc(nr); un.alloc(nr); v.alloc(nd); vn.alloc(nd); w.alloc(nd);
    scale_copy<T>(nr, 1.0 / beta1, b, u.p, d.s);
    d.atb(u.p, v.p);
    double alpha = std::sqrt(d.nrm2sq(v.p, nd, false));
    if (!(alpha > 0.0)) fail(CTK_E_DEGENERATE, "lsqr: A^T b vanished");
    scal<T>(nd, 1.0 / alpha, v.p, d.s);
    CTK_CUDA(cudaMemcpyAsync(w.p, v.p, sizeof(T) * nd, cudaMemcpyDeviceToDevice, d.s));
    fill<T>(nd, T(0), x, d.s);
    double phibar = beta1, rhobar = alpha;
    int k = 0;
    while (k < o.max_iters) {
        ++k;
        d.ax(v.p, un.p);
        double beta = std::sqrt(d.axpy_n2(-alpha, u.p, un.p, nr, true));
        bool down = beta <= tol;
        if (beta > 0.0) {
            scal<T>(nr, 1.0 / beta, un.p, d.s);
            std::swap(u.p, un.p);
            d.atb(u.p, vn.p);
            alpha = std::sqrt(d.axpy_n2(-beta, v.p, vn.p, nd, false));
            if (alpha > 0.0) {
                scal<T>(nd, 1.0 / alpha, vn.p, d.s);
                std::swap(v.p, vn.p);
            }
            down = down || alpha <= tol;
        } else {
            alpha = 0.0;
        }
        const double rho = std::sqrt(rhobar * rhobar + beta * beta);
        const double c = rhobar / rho, sn = beta / rho;
        const double theta = sn * alpha;
        rhobar = -c * alpha;
        const double phi = c * phibar;
        phibar = sn * phibar;
        lsqr_update<T>(nd, phi / rho, theta / rho, x, w.p, v.p, d.s);
        if (k < o.max_iters && !down) d.announce_ax(v.p, un.p);
        if (mon.record(k, x, phibar / beta1)) break;
        if (down) {
            mon.reason = CTK_STOP_BREAKDOWN;
            break;
        }
    }
    mon.finish(k);
}

template <class T>
void lsmr(Dev<T>& d, const T* b, double lambda, const ctk_solver_opts& o, T* x, ctk_solve_log* log) {
    Geometry& g = d.g;
    const size_t nd = g.domain(), nr = g.range();
    if (lambda < 0.0) fail(CTK_E_PARAMETER, "lsmr: lambda must be nonnegative");
    Monitor<T> mon(d, b, o, log, "lsmr");
    const double damp = lambda;
    const double beta1 = mon.bnorm;
    const double tol = breakdown_factor<T>() * beta1;
    Vec<T> u, un, v, vn, h, hbar;
    u.alloc(nr); un.alloc(nr); v.alloc(nd); vn.alloc(nd); h.alloc(nd); hbar.alloc(nd);
    scale_copy<T>(nr, 1.0 / beta1, b, u.p, d.s);
    d.atb(u.p, v.p);
    double alpha = std::sqrt(d.nrm2sq(v.p, nd, false));
    if (!(alpha > 0.0)) fail(CTK_E_DEGENERATE, "lsmr: A^T b vanished");
    scal<T>(nd, 1.0 / alpha, v.p, d.s);
    double zetabar = alpha * beta1, alphabar = alpha;
    double rho = 1, rhobar = 1, cbar = 1, sbar = 0;
    CTK_CUDA(cudaMemcpyAsync(h.p, v.p, sizeof(T) * nd, cudaMemcpyDeviceToDevice, d.s));
    fill<T>(nd, T(0), hbar.p, d.s);
    fill<T>(nd, T(0), x, d.s);
    double betadd = beta1, betad = 0, rhodold = 1, tautildeold = 0, thetatilde = 0, zeta = 0, dsq = 0;
    int k = 0;
    while (k < o.max_iters) {
        ++k;
        d.ax(v.p, un.p);
        double beta = std::sqrt(d.axpy_n2(-alpha, u.p, un.p, nr, true));
        bool down = beta <= tol;
        if (beta > 0.0) {
            scal<T>(nr, 1.0 / beta, un.p, d.s);
            std::swap(u.p, un.p);
            d.atb(u.p, vn.p);
            alpha = std::sqrt(d.axpy_n2(-beta, v.p, vn.p, nd, false));
            if (alpha > 0.0) {
                scal<T>(nd, 1.0 / alpha, vn.p, d.s);
                std::swap(v.p, vn.p);
            }
            down = down || alpha <= tol;
        } else {
            alpha = 0.0;
        }
        const double alphahat = std::sqrt(alphabar * alphabar + damp * damp);
        const double chat = alphabar / alphahat, shat = damp / alphahat;
        const double rhoold = rho;
        rho = std::sqrt(alphahat * alphahat + beta * beta);
        const double c = alphahat / rho, sn = beta / rho;
        const double thetanew = sn * alpha;
        alphabar = c * alpha;
        const double rhobarold = rhobar, zetaold = zeta;
        const double thetabar = sbar * rho;
        const double rhotemp = cbar * rho;
        rhobar = std::sqrt(rhotemp * rhotemp + thetanew * thetanew);
        cbar = rhotemp / rhobar;
        sbar = thetanew / rhobar;
        zeta = cbar * zetabar;
        zetabar = -sbar * zetabar;
        lsmr_update<T>(nd, thetabar * rho / (rhoold * rhobarold), zeta / (rho * rhobar), thetanew / rho, x, h.p, hbar.p,
                       v.p, d.s);
        const double betaacute = chat * betadd;
        const double betacheck = -shat * betadd;
        const double betahat = c * betaacute;
        betadd = -sn * betaacute;
        const double thetatildeold = thetatilde;
        const double rhotildeold = std::sqrt(rhodold * rhodold + thetabar * thetabar);
        const double ctildeold = rhodold / rhotildeold, stildeold = thetabar / rhotildeold;
        thetatilde = stildeold * rhobar;
        rhodold = ctildeold * rhobar;
        betad = -stildeold * betad + ctildeold * betahat;
        tautildeold = (zetaold - thetatildeold * tautildeold) / rhotildeold;
        const double taud = (zeta - thetatilde * tautildeold) / rhodold;
        dsq += betacheck * betacheck;
        const double normr = std::sqrt(dsq + (betad - taud) * (betad - taud) + betadd * betadd);
        if (k < o.max_iters && !down) d.announce_ax(v.p, un.p);
        if (mon.record(k, x, normr / beta1, true, lambda)) break;
        if (down) {
            mon.reason = CTK_STOP_BREAKDOWN;
            break;
        }
    }
    mon.finish(k);
}

// CGS2 against the first m stored basis vectors (krylov.hpp:21-31); range bases are
// sharded across ranks, so their coefficients are summed over ranks.
template <class T>
void cgs2(Dev<T>& d, const T* basis, size_t ld, int m, T* wv, size_t n, bool range, double* d_coef, double* scratch) {
    for (int pass = 0; pass < 2; ++pass) {
        block_dot<T>(n, m, basis, ld, wv, d_coef, scratch, d.s);
        if (d.sharded(range)) comm_sum_vector(d.g.comm, d_coef, m, d.s);  // one gather per pass
        block_axpy<T>(n, m, -1.0, d_coef, basis, ld, wv, d.s);
    }
}

template <class T>
void hybrid_lsqr(Dev<T>& d, const T* b, const ctk_hybrid_strategy& strat, const ctk_solver_opts& o, T* x,
                 ctk_solve_log* log) {
    Geometry& g = d.g;
    const size_t nd = g.domain(), nr = g.range();
    if (strat.kind == CTK_LAMBDA_FIXED && strat.lambda < 0.0) fail(CTK_E_PARAMETER, "fixed lambda must be nonnegative");
    if (strat.kind == CTK_LAMBDA_DP && !(strat.noise_level > 0.0 && strat.noise_level < 1.0))
        fail(CTK_E_PARAMETER, "dp strategy needs a noise level in (0,1)");
    if (strat.kind < 0 || strat.kind > 2) fail(CTK_E_PARAMETER, "unknown lambda strategy");
    Monitor<T> mon(d, b, o, log, "hybrid_lsqr");
    const int cap = o.max_iters + 2;
    DevBuf &Ub = pooled(), &Vb = pooled(), &coefb = pooled(), &scratchb = pooled();
    Ub.ensure(sizeof(T) * nr * size_t(cap));
    Vb.ensure(sizeof(T) * nd * size_t(cap));
    coefb.ensure(sizeof(double) * size_t(cap));
    scratchb.ensure(sizeof(double) * size_t(cap) * kRedBlocks);
    T* U = Ub.as<T>();
    T* V = Vb.as<T>();
    auto Ui = [&](int i) { return U + size_t(i) * nr; };
    auto Vi = [&](int i) { return V + size_t(i) * nd; };
    // gk_init (krylov.hpp:50-67)
    const double beta1 = mon.bnorm;
    const double tol = breakdown_factor<T>() * beta1;
    scale_copy<T>(nr, 1.0 / beta1, b, Ui(0), d.s);
    d.atb(Ui(0), Vi(0));
    const double alpha1 = std::sqrt(d.nrm2sq(Vi(0), nd, false));
    if (!(alpha1 > 0.0)) fail(CTK_E_DEGENERATE, "gk_init: B u_1 vanished");
    scal<T>(nd, 1.0 / alpha1, Vi(0), d.s);
    int nu_ = 1, nv_ = 1;
    std::vector<double> alphas{alpha1}, betas;
    Vec<T> ynum;
    DevBuf& dy = pooled();
    dy.ensure(sizeof(double) * size_t(cap));
    int k = 0;
    while (k < o.max_iters) {
        // gk_expand (krylov.hpp:69-92)
        bool breakdown = false;
        {
            const int j = nv_;
            T* wv = Ui(nu_);
            d.ax(Vi(j - 1), wv);
            axpy<T>(nr, -alphas[size_t(j - 1)], Ui(j - 1), wv, d.s);
            if (o.reorth) cgs2<T>(d, U, nr, nu_, wv, nr, true, coefb.as<double>(), scratchb.as<double>());
            const double beta = std::sqrt(d.nrm2sq(wv, nr, true));
            if (beta <= tol) {
                breakdown = true;
            } else {
                scal<T>(nr, 1.0 / beta, wv, d.s);
                ++nu_;
                betas.push_back(beta);
                T* z = Vi(nv_);
                d.atb(Ui(j), z);
                axpy<T>(nd, -beta, Vi(j - 1), z, d.s);
                if (o.reorth) cgs2<T>(d, V, nd, nv_, z, nd, false, coefb.as<double>(), scratchb.as<double>());
                const double alpha = std::sqrt(d.nrm2sq(z, nd, false));
                if (alpha <= tol) {
                    breakdown = true;
                } else {
                    scal<T>(nd, 1.0 / alpha, z, d.s);
                    ++nv_;
                    alphas.push_back(alpha);
                }
            }
        }
        if (breakdown && int(betas.size()) < k + 1) {
            mon.reason = CTK_STOP_BREAKDOWN;
            break;
        }
        ++k;
        std::vector<double> H(size_t(k + 1) * k, 0.0);
        for (int jj = 0; jj < k; ++jj) {
            H[size_t(jj) * k + jj] = alphas[size_t(jj)];
            H[size_t(jj + 1) * k + jj] = betas[size_t(jj)];
        }
        const double lambda_k = choose_lambda(strat, H, k, beta1);
        double fit = 0.0;
        const std::vector<double> y = projected_tikhonov(H, k, beta1, lambda_k, &fit);
        // basis_combination (gmres.hpp:33-39): x = sum_i T(y_i) V_i, accumulated in order
        CTK_CUDA(cudaMemcpyAsync(dy.p, y.data(), sizeof(double) * y.size(), cudaMemcpyHostToDevice, d.s));
        fill<T>(nd, T(0), x, d.s);
        block_axpy<T>(nd, int(y.size()), 1.0, dy.as<double>(), V, nd, x, d.s);
        CTK_CUDA(cudaStreamSynchronize(d.s));  // y (host) must outlive the async copy
        if (k < o.max_iters && !breakdown) d.announce_ax(Vi(nv_ - 1), Ui(nu_));
        if (mon.record(k, x, fit / beta1, true, lambda_k)) break;
        if (breakdown) {
            mon.reason = CTK_STOP_BREAKDOWN;
            break;
        }
    }
    mon.finish(k);
    log->stored_domain_basis = nv_;
    log->stored_range_basis = nu_;
}

// stacked operator K = [A; lam diag(w) D] of stack_weighted_gradient
template <class T>
struct Stacked {
    Dev<T>& d;
    const T* w;
    double lam;
    size_t nd, nr;
    void fwd(const T* x, T* y) {
        d.ax(x, y);
        const T* above = d.slice_above(x);
        gradient_scaled<T>(d.g.nx, d.g.ny, d.g.nz_local(), x, w, lam, y + nr, y + nr + nd, y + nr + 2 * nd, d.s, above);
    }
    void back(const T* y, T* x) {
        d.atb(y, x);
        const T* below = d.weighted_slice_below(y + nr + 2 * nd, w, lam);
        gradient_adjoint_scaled_add<T>(d.g.nx, d.g.ny, d.g.nz_local(), y + nr, y + nr + nd, y + nr + 2 * nd, w, lam, x,
                                       d.s, below, d.slab_mode() && !d.last_slab());
    }
    // squared norm of a stacked vector: sharded range part + replicated gradient part
    double n2(const T* y) { return d.nrm2sq(y, nr, true) + d.nrm2sq(y + nr, 3 * nd, false); }
    double axpy_n2(double a, const T* x, T* y) { return d.axpy_n2(a, x, y, nr, true) + d.axpy_n2(a, x + nr, y + nr, 3 * nd, false); }
};

template <class T>
void cgls_tv(Dev<T>& d, const T* b, double lambda, int outer_iters, int inner_iters, bool warm,
             const ctk_solver_opts& o, T* x, ctk_solve_log* log) {
    Geometry& g = d.g;
    const size_t nd = g.domain(), nr = g.range();
    if (!(lambda > 0.0)) fail(CTK_E_PARAMETER, "cgls_tv: lambda must be positive");
    if (outer_iters < 1 || inner_iters < 1) fail(CTK_E_PARAMETER, "cgls_tv: outer and inner iteration counts must be >= 1");
    Monitor<T> mon(d, b, o, log, "cgls_tv");
    const size_t ns = nr + 3 * nd;
    Vec<T> wts, r, s, p, q;
    wts.alloc(nd); r.alloc(ns); s.alloc(nd); p.alloc(nd); q.alloc(ns);
    fill<T>(nd, T(0), x, d.s);
    int k = 0;
    bool stopped = false;
    log->n_outer_starts = 0;
    for (int outer = 0; outer < outer_iters && !stopped; ++outer) {
        // tv_weights (tv.hpp:28-43): eps = 1e-4 max|x|
        reduce_absmax<T>(nd, x, d.w.results, d.w, d.s);
        const double eps = 1e-4 * d.domain_max(d.fetch(0));
        tv_weights<T>(g.nx, g.ny, g.nz_local(), x, eps, wts.p, d.s, d.slice_above(x));
        Stacked<T> K{d, wts.p, lambda, nd, nr};
        // rhs = [b; 0]
        if (log->outer_starts) log->outer_starts[log->n_outer_starts++] = k;
        mon.have_prev = false;  // reset_increase_baseline
        if (!warm) fill<T>(nd, T(0), x, d.s);
        CTK_CUDA(cudaMemcpyAsync(r.p, b, sizeof(T) * nr, cudaMemcpyDeviceToDevice, d.s));
        fill<T>(3 * nd, T(0), r.p + nr, d.s);
        const double rhs_norm = std::sqrt(K.n2(r.p));
        if (warm) {
            K.fwd(x, q.p);
            axpy<T>(ns, -1.0, q.p, r.p, d.s);
        }
        K.back(r.p, s.p);
        CTK_CUDA(cudaMemcpyAsync(p.p, s.p, sizeof(T) * nd, cudaMemcpyDeviceToDevice, d.s));
        double gamma = d.nrm2sq(s.p, nd, false);
        for (int inner = 0; inner < inner_iters; ++inner) {
            if (!(gamma > 0.0)) break;
            K.fwd(p.p, q.p);
            const double delta = K.n2(q.p);
            if (!(delta > 0.0)) break;
            const double alpha = gamma / delta;
            axpy<T>(nd, alpha, p.p, x, d.s);
            const double rr = K.axpy_n2(-alpha, q.p, r.p);
            ++k;
            auto advance = [&] {
                K.back(r.p, s.p);
                const double gnew = d.nrm2sq(s.p, nd, false);
                const double beta = gnew / gamma;
                gamma = gnew;
                xpby<T>(nd, s.p, beta, p.p, d.s);
            };
            const bool ahead = inner + 1 < inner_iters && d.can_pair();  // as cgls: pair A x with the next A p
            if (ahead) {
                advance();
                d.announce_ax(p.p, q.p);
            }
            if (mon.record(k, x, std::sqrt(rr) / rhs_norm, true, lambda)) {
                stopped = true;
                break;
            }
            if (!ahead) advance();
        }
    }
    mon.finish(k);
}

// SIRT (solvers.hpp:233-287): x <- x + C B (R (b - A x)), R and C the inverse row / column
// sums of the pair (A 1, B 1) floored at 1e-6 of their maximum.  One genuine forward per
// iteration drives both the update and the logged residual.
template <class T>
void sirt(Dev<T>& d, const T* b, const ctk_solver_opts& o, T* x, ctk_solve_log* log) {
    Geometry& g = d.g;
    const size_t nd = g.domain(), nr = g.range();
    log->iterations = log->n_relative_error = log->n_lambda = log->n_warnings = 0;
    if (!(std::sqrt(d.nrm2sq(b, nr, true)) > 0.0)) {
        // zero data: x = 0 is already the fixed point (solvers.hpp:240-251)
        fill<T>(nd, T(0), x, d.s);
        log->iterations_run = 0;
        log->stop_reason = CTK_STOP_TOLERANCE;
        return;
    }
    Monitor<T> mon(d, b, o, log, "sirt");
    Vec<T> row_inv, col_inv, r, corr, ax;
    row_inv.alloc(nr); col_inv.alloc(nd); r.alloc(nr); corr.alloc(nd); ax.alloc(nr);
    // inverse weights from the pair applied to all-ones vectors (solvers.hpp:257-267)
    auto inverse_weights = [&](T* w, size_t n, bool range) {
        reduce_absmax<T>(n, w, d.w.results, d.w, d.s);
        double wmax = d.fetch(0);
        if (d.sharded(range)) wmax = comm_max_scalar(g.comm, wmax);
        if (!(T(wmax) > T(0))) fail(CTK_E_DEGENERATE, "sirt: operator maps ones to zero");
        inv_floor<T>(n, double(T(1e-6) * T(wmax)), w, d.s);
    };
    fill<T>(nd, T(1), corr.p, d.s);
    d.ax(corr.p, row_inv.p);
    inverse_weights(row_inv.p, nr, true);
    fill<T>(nr, T(1), r.p, d.s);
    d.atb(r.p, col_inv.p);
    inverse_weights(col_inv.p, nd, false);
    fill<T>(nd, T(0), x, d.s);
    CTK_CUDA(cudaMemcpyAsync(r.p, b, sizeof(T) * nr, cudaMemcpyDeviceToDevice, d.s));  // b - A x for x = 0
    int k = 0;
    while (k < o.max_iters) {
        ++k;
        mul<T>(nr, row_inv.p, r.p, ax.p, d.s);  // scaled = R r (ax is scratch here)
        d.atb(ax.p, corr.p);
        add_mul<T>(nd, col_inv.p, corr.p, x, d.s);
        d.ax(x, ax.p);
        sub_nrm2sq<T>(nr, b, ax.p, r.p, d.w.results, d.w, d.s);
        const double expl = std::sqrt(d.part_sum(d.fetch(0), true)) / mon.bnorm;
        if (mon.record(k, x, expl, false, 0.0, &expl)) break;
    }
    mon.finish(k);
}

// AB-GMRES (ab = true: Arnoldi on A B over the range, x = B u) and BA-GMRES (Arnoldi on
// B A over the domain with right-hand side B b), gmres.hpp:41-114; Arnoldi with modified
// Gram-Schmidt plus an optional classical second pass (krylov.hpp:94-145).  x is rebuilt
// from the whole basis every iteration like the reference (basis_combination).
template <class T>
void abba_gmres(Dev<T>& d, const T* b, const ctk_solver_opts& o, T* x, ctk_solve_log* log, bool ab) {
    Geometry& g = d.g;
    const size_t nd = g.domain(), nr = g.range();
    const size_t n = ab ? nr : nd;  // Arnoldi space
    Monitor<T> mon(d, b, o, log, ab ? "ab_gmres" : "ba_gmres");
    const int cap = o.max_iters + 1;
    DevBuf &Wb = pooled(), &dyb = pooled();
    Wb.ensure(sizeof(T) * n * size_t(cap));
    dyb.ensure(sizeof(double) * size_t(cap));
    T* W = Wb.as<T>();
    auto Wi = [&](int i) { return W + size_t(i) * n; };
    Vec<T> tmp, u;
    tmp.alloc(ab ? nd : nr);  // the intermediate of the squared operator
    if (ab) u.alloc(nr);
    auto apply_square = [&](const T* in, T* out) {
        if (ab) {
            d.atb(in, tmp.p);
            d.ax(tmp.p, out);
        } else {
            d.ax(in, tmp.p);
            d.atb(tmp.p, out);
        }
    };
    // arnoldi_init (krylov.hpp:107-117)
    if (ab) CTK_CUDA(cudaMemcpyAsync(Wi(0), b, sizeof(T) * nr, cudaMemcpyDeviceToDevice, d.s));
    else d.atb(b, Wi(0));
    const double beta1 = std::sqrt(d.nrm2sq(Wi(0), n, ab));
    if (!(beta1 > 0.0)) fail(CTK_E_DEGENERATE, "arnoldi_init: zero right-hand side");
    scal<T>(n, 1.0 / beta1, Wi(0), d.s);
    const double tol = breakdown_factor<T>() * beta1;
    std::vector<std::vector<double>> hcols;
    int nbasis = 1;
    int k = 0;
    while (k < o.max_iters) {
        ++k;
        // arnoldi_expand (krylov.hpp:119-145)
        const int j = int(hcols.size());
        T* w = Wi(j + 1);
        apply_square(Wi(j), w);
        std::vector<double> h(size_t(j + 2), 0.0);
        for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt, in order
            reduce_dot<T>(n, Wi(i), w, d.w.results, d.w, d.s);
            double hi = d.fetch(0);
            hi = d.part_sum(hi, ab);
            h[size_t(i)] = double(T(hi));
            axpy<T>(n, -h[size_t(i)], Wi(i), w, d.s);
        }
        if (o.reorth) {
            for (int i = 0; i <= j; ++i) {
                reduce_dot<T>(n, Wi(i), w, d.w.results, d.w, d.s);
                double c = d.fetch(0);
                c = d.part_sum(c, ab);
                c = double(T(c));
                axpy<T>(n, -c, Wi(i), w, d.s);
                h[size_t(i)] = double(T(h[size_t(i)]) + T(c));
            }
        }
        const double hnext = double(T(std::sqrt(d.nrm2sq(w, n, ab))));
        h[size_t(j + 1)] = hnext;
        hcols.push_back(h);
        const bool breakdown = hnext <= tol;
        if (!breakdown) {
            scal<T>(n, 1.0 / hnext, w, d.s);
            ++nbasis;
        }
        // projected least squares on the (k+1) x k Hessenberg (gmres.hpp:14-31)
        std::vector<double> H(size_t(k + 1) * k, 0.0);
        for (int c = 0; c < k; ++c)
            for (int r = 0; r < int(hcols[size_t(c)].size()) && r <= k; ++r) H[size_t(r) * k + c] = hcols[size_t(c)][size_t(r)];
        double resid = 0.0;
        const std::vector<double> y = projected_ls(H, k, beta1, &resid);
        // basis_combination (gmres.hpp:33-39) over the first k basis vectors
        CTK_CUDA(cudaMemcpyAsync(dyb.p, y.data(), sizeof(double) * y.size(), cudaMemcpyHostToDevice, d.s));
        T* comb = ab ? u.p : x;
        fill<T>(n, T(0), comb, d.s);
        block_axpy<T>(n, k, 1.0, dyb.as<double>(), W, n, comb, d.s);
        CTK_CUDA(cudaStreamSynchronize(d.s));  // y (host) must outlive the async copy
        if (ab) d.atb(u.p, x);
        if (mon.record(k, x, resid / beta1)) break;
        if (breakdown) {
            mon.reason = CTK_STOP_BREAKDOWN;
            break;
        }
    }
    mon.finish(k);
    log->stored_domain_basis = ab ? 0 : nbasis;
    log->stored_range_basis = ab ? nbasis : 0;
}

// Flexible hybrid LSQR with TV priorconditioning (hybrid.hpp:118-168, tv.hpp:112-185,
// krylov.hpp:147-224): flexible Golub-Kahan A Z_k = U_{k+1} M_k where z_j = P_j v_j and P_j
// is an inner CG solve of (D^T diag(w^2) D + tau^2 I) z = v with IRN weights w from the
// current iterate (tau = 1e-3 lambda0, <= 50 CG steps to 1e-6); modified Gram-Schmidt
// (+ a classical pass when reorth) on U, full re-orthogonalisation of V; projected
// Tikhonov on the (k+1) x k Hessenberg M with lambda fixed or by GCV; x = Z_k y.
template <class T>
void flsqr_tv(Dev<T>& d, const T* b, const ctk_hybrid_strategy& strat, const ctk_solver_opts& o, T* x,
              ctk_solve_log* log) {
    Geometry& g = d.g;
    const size_t nd = g.domain(), nr = g.range();
    if (strat.kind == CTK_LAMBDA_DP) fail(CTK_E_PARAMETER, "flsqr_tv: dp strategy is not supported, use fixed or gcv");
    if (strat.kind != CTK_LAMBDA_FIXED && strat.kind != CTK_LAMBDA_GCV) fail(CTK_E_PARAMETER, "unknown lambda strategy");
    if (strat.kind == CTK_LAMBDA_FIXED && strat.lambda < 0.0) fail(CTK_E_PARAMETER, "fixed lambda must be nonnegative");
    const double lambda0 = strat.kind == CTK_LAMBDA_FIXED && strat.lambda > 0.0 ? strat.lambda : 1.0;
    const double tau = 1e-3 * lambda0;
    const T tau2 = T(tau * tau);
    constexpr int kMaxInner = 50;
    constexpr double kInnerTol = 1e-6;
    Monitor<T> mon(d, b, o, log, "flsqr_tv");
    log->n_warnings = 0;
    const int cap = o.max_iters + 2;
    DevBuf &Ub = pooled(), &Vb = pooled(), &Zb = pooled(), &coefb = pooled();
    Ub.ensure(sizeof(T) * nr * size_t(cap));
    Vb.ensure(sizeof(T) * nd * size_t(cap));
    Zb.ensure(sizeof(T) * nd * size_t(cap));
    coefb.ensure(sizeof(double) * size_t(cap));
    auto Ui = [&](int i) { return Ub.as<T>() + size_t(i) * nr; };
    auto Vi = [&](int i) { return Vb.as<T>() + size_t(i) * nd; };
    auto Zi = [&](int i) { return Zb.as<T>() + size_t(i) * nd; };
    Vec<T> w2, r, p, ap, gx, gy, gz;
    w2.alloc(nd); r.alloc(nd); p.alloc(nd); ap.alloc(nd); gx.alloc(nd); gy.alloc(nd); gz.alloc(nd);
    // flexible_gk_init (krylov.hpp:161-177)
    const double beta1 = mon.bnorm;
    const double tol = breakdown_factor<T>() * beta1;
    scale_copy<T>(nr, 1.0 / beta1, b, Ui(0), d.s);
    d.atb(Ui(0), Vi(0));
    const double nv0 = std::sqrt(d.nrm2sq(Vi(0), nd, false));
    if (!(nv0 > 0.0)) fail(CTK_E_DEGENERATE, "flexible_gk_init: B u_1 vanished");
    scal<T>(nd, 1.0 / nv0, Vi(0), d.s);
    int nu_ = 1, nv_ = 1, nz_ = 0;
    std::vector<std::vector<double>> mcols;
    fill<T>(nd, T(0), x, d.s);
    // the TV operator D^T diag(w^2) D + tau^2 I of the preconditioner (tv.hpp:134-143)
    auto apply_tv = [&](const T* in, T* out) {
        scale_copy<T>(nd, double(tau2), in, out, d.s);
        gradient_scaled<T>(g.nx, g.ny, g.nz_local(), in, w2.p, 1.0, gx.p, gy.p, gz.p, d.s, d.slice_above(in));
        const T* below = d.weighted_slice_below(gz.p, nullptr, 1.0);
        gradient_adjoint_scaled_add<T>(g.nx, g.ny, g.nz_local(), gx.p, gy.p, gz.p, nullptr, 1.0, out, d.s, below,
                                       d.slab_mode() && !d.last_slab());
    };
    // inner CG from zero on the SPD system (tv.hpp:145-168); returns false if not converged
    auto precond = [&](const T* v, T* z) {
        fill<T>(nd, T(0), z, d.s);
        CTK_CUDA(cudaMemcpyAsync(r.p, v, sizeof(T) * nd, cudaMemcpyDeviceToDevice, d.s));
        CTK_CUDA(cudaMemcpyAsync(p.p, v, sizeof(T) * nd, cudaMemcpyDeviceToDevice, d.s));
        double rr = d.nrm2sq(r.p, nd, false);
        const double target = kInnerTol * std::sqrt(rr);
        bool converged = !(std::sqrt(rr) > 0.0);
        for (int it = 0; it < kMaxInner && !converged; ++it) {
            apply_tv(p.p, ap.p);
            reduce_dot<T>(nd, p.p, ap.p, d.w.results, d.w, d.s);
            const double pap = d.part_sum(d.fetch(0), false);
            if (!(pap > 0.0)) break;
            const double alpha = rr / pap;
            axpy<T>(nd, alpha, p.p, z, d.s);
            const double rr_new = d.axpy_n2(-alpha, ap.p, r.p, nd, false);
            if (std::sqrt(rr_new) <= target) {
                converged = true;
                break;
            }
            const double beta = rr_new / rr;
            rr = rr_new;
            xpby<T>(nd, r.p, beta, p.p, d.s);
        }
        return converged;
    };
    // modified Gram-Schmidt of w against the first m vectors of a basis, in order
    auto mgs = [&](auto basis, int m, T* wv, size_t n, bool range, std::vector<double>* coef) {
        for (int i = 0; i < m; ++i) {
            reduce_dot<T>(n, basis(i), wv, d.w.results, d.w, d.s);
            const double c = double(T(d.part_sum(d.fetch(0), range)));
            axpy<T>(n, -c, basis(i), wv, d.s);
            if (coef) (*coef)[size_t(i)] = double(T((*coef)[size_t(i)]) + T(c));
        }
    };
    int k = 0;
    while (k < o.max_iters) {
        // the preconditioner of iteration k+1, from the current iterate: w^2 of tv_weights
        reduce_absmax<T>(nd, x, d.w.results, d.w, d.s);
        const double eps = 1e-4 * d.domain_max(d.fetch(0));
        tv_weights<T>(g.nx, g.ny, g.nz_local(), x, eps, w2.p, d.s, d.slice_above(x));
        mul<T>(nd, w2.p, w2.p, w2.p, d.s);
        // flexible_gk_expand (krylov.hpp:179-223)
        bool breakdown = false;
        {
            const int j = int(mcols.size());
            T* z = Zi(j);
            if (!precond(Vi(j), z) && log->warning_iterations && log->n_warnings < log->capacity)
                log->warning_iterations[log->n_warnings++] = k + 1;
            if (!(std::sqrt(d.nrm2sq(z, nd, false)) > 0.0)) {
                breakdown = true;
            } else {
                T* wv = Ui(nu_);
                d.ax(z, wv);
                std::vector<double> m(size_t(j + 2), 0.0);
                mgs(Ui, j + 1, wv, nr, true, &m);
                if (o.reorth) mgs(Ui, j + 1, wv, nr, true, &m);
                const double mnext = double(T(std::sqrt(d.nrm2sq(wv, nr, true))));
                m[size_t(j + 1)] = mnext;
                ++nz_;
                mcols.push_back(m);
                if (mnext <= tol) {
                    breakdown = true;
                } else {
                    scal<T>(nr, 1.0 / mnext, wv, d.s);
                    ++nu_;
                    T* v = Vi(nv_);
                    d.atb(wv, v);
                    for (int pass = 0; pass < (o.reorth ? 2 : 1); ++pass) mgs(Vi, nv_, v, nd, false, nullptr);
                    const double nvn = std::sqrt(d.nrm2sq(v, nd, false));
                    if (nvn <= tol) {
                        breakdown = true;
                    } else {
                        scal<T>(nd, 1.0 / nvn, v, d.s);
                        ++nv_;
                    }
                }
            }
        }
        if (breakdown && int(mcols.size()) < k + 1) {
            mon.reason = CTK_STOP_BREAKDOWN;
            break;
        }
        ++k;
        std::vector<double> M(size_t(k + 1) * k, 0.0);
        for (int c = 0; c < k; ++c)
            for (int rr = 0; rr < int(mcols[size_t(c)].size()) && rr <= k; ++rr)
                M[size_t(rr) * k + c] = mcols[size_t(c)][size_t(rr)];
        const double lambda_k = choose_lambda(strat, M, k, beta1);
        double fit = 0.0;
        const std::vector<double> y = projected_tikhonov(M, k, beta1, lambda_k, &fit);
        CTK_CUDA(cudaMemcpyAsync(coefb.p, y.data(), sizeof(double) * y.size(), cudaMemcpyHostToDevice, d.s));
        fill<T>(nd, T(0), x, d.s);
        block_axpy<T>(nd, int(y.size()), 1.0, coefb.as<double>(), Zb.as<T>(), nd, x, d.s);
        CTK_CUDA(cudaStreamSynchronize(d.s));  // y (host) must outlive the async copy
        if (k < o.max_iters && !breakdown) d.announce_ax(Vi(nv_ - 1), Ui(nu_));
        if (mon.record(k, x, fit / beta1, true, lambda_k)) break;
        if (breakdown) {
            mon.reason = CTK_STOP_BREAKDOWN;
            break;
        }
    }
    mon.finish(k);
    log->stored_domain_basis = nz_;
    log->stored_range_basis = nu_;
}

}  // namespace

template <class T>
void solve_device(Geometry& g, int solver, int variant, const T* d_b, double lambda, const ctk_hybrid_strategy* st,
                  int outer, int inner, int warm, const ctk_solver_opts* o, T* d_x, ctk_solve_log* log) {
    g.require_angles();
    if (variant != CTK_BP_MATCHED && variant != CTK_BP_VOXEL_DRIVEN) fail(CTK_E_PARAMETER, "unknown backprojector variant");
    const int need = solver == 4 ? std::max(1, outer) * std::max(1, inner) : (o ? o->max_iters : 0);
    validate_opts(o, log, need);
    struct PoolScope {  // hand out this handle's workspace slots from the start
        explicit PoolScope(Geometry& gg) { gg.ws_next = 0; t_pool = &gg; }
        ~PoolScope() { t_pool = nullptr; }
    } pool_scope(g);
    Dev<T> d(g, variant);
    switch (solver) {
        case 0: cgls<T>(d, d_b, *o, d_x, log); break;
        case 1: lsqr<T>(d, d_b, *o, d_x, log); break;
        case 2: lsmr<T>(d, d_b, lambda, *o, d_x, log); break;
        case 3:
            if (!st) fail(CTK_E_PARAMETER, "hybrid_lsqr needs a strategy");
            hybrid_lsqr<T>(d, d_b, *st, *o, d_x, log);
            break;
        case 4: cgls_tv<T>(d, d_b, lambda, outer, inner, warm != 0, *o, d_x, log); break;
        case 5: sirt<T>(d, d_b, *o, d_x, log); break;
        case 6: abba_gmres<T>(d, d_b, *o, d_x, log, true); break;
        case 7: abba_gmres<T>(d, d_b, *o, d_x, log, false); break;
        case 8:
            if (!st) fail(CTK_E_PARAMETER, "flsqr_tv needs a strategy");
            flsqr_tv<T>(d, d_b, *st, *o, d_x, log);
            break;
        default: fail(CTK_E_PARAMETER, "unknown solver");
    }
    CTK_CUDA(cudaStreamSynchronize(g.stream));
}

template void solve_device<float>(Geometry&, int, int, const float*, double, const ctk_hybrid_strategy*, int, int, int,
                                  const ctk_solver_opts*, float*, ctk_solve_log*);
template void solve_device<double>(Geometry&, int, int, const double*, double, const ctk_hybrid_strategy*, int, int,
                                   int, const ctk_solver_opts*, double*, ctk_solve_log*);

}  // namespace ctkb
