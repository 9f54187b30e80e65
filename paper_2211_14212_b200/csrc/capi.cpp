// extern "C" surface of libctk_b200.so (include/ctk_b200.h).  Every entry point catches
// the internal exceptions and returns the status of the reference's error taxonomy
// (types.hpp:14-31); the message is kept thread-locally for ctk_last_error.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "ctk_internal.h"
#include "regparam.h"

namespace ctkb {
void geometry_validate(const ctk_geom_desc* d);  // ConeGeometry::validate, no device work
Geometry* geometry_create(const ctk_geom_desc* d);
void nccl_unique_id(void* out128);
Comm* comm_create_nccl(const void* id128, int nranks, int rank);
Comm* comm_adopt_nccl(void* nccl_comm, int nranks, int rank);
void comm_destroy(Comm* c);
template <class T>
void solve_device(Geometry& g, int solver, int variant, const T* d_b, double lambda, const ctk_hybrid_strategy* st,
                  int outer, int inner, int warm, const ctk_solver_opts* o, T* d_x, ctk_solve_log* log);
}  // namespace ctkb

// ctk_geom / ctk_comm stay incomplete: the handles are ctkb::Geometry* / ctkb::Comm*.
namespace {

thread_local std::string t_msg;
thread_local int t_code = 0;
thread_local int t_iter = 0;

template <class F>
int guard(F&& f) {
    try {
        f();
        return CTK_OK;
    } catch (const ctkb::Error& e) {
        t_msg = e.what();
        t_code = e.code;
        t_iter = e.iteration;
        return e.code;
    } catch (const std::bad_alloc&) {
        t_msg = "host allocation failed";
        t_code = CTK_E_PARAMETER;
        return t_code;
    } catch (const std::exception& e) {
        t_msg = e.what();
        t_code = CTK_E_PARAMETER;
        return t_code;
    }
}

ctkb::Geometry& G(const ctk_geom* g) {
    if (!g) ctkb::fail(CTK_E_PARAMETER, "null geometry handle");
    return *reinterpret_cast<ctkb::Geometry*>(const_cast<ctk_geom*>(g));
}

// Device-pointer entry points follow the CUDA convention: the caller's stream, NULL = the
// legacy default stream (so work is ordered with the caller's default-stream producers).
cudaStream_t S(ctkb::Geometry&, void* stream) { return static_cast<cudaStream_t>(stream); }

void check_variant(int v) {
    if (v != CTK_BP_MATCHED && v != CTK_BP_VOXEL_DRIVEN) ctkb::fail(CTK_E_PARAMETER, "unknown backprojector variant");
}

// With a communicator attached the public operators follow the solvers' rule (solvers.cpp
// Dev::ax / Dev::atb): under angle sharding A x is local and every A^T b partial volume is
// summed; under z-slab sharding A x = sum_r A x_r is summed and A^T b is local.
template <class T>
void ax_dev(ctkb::Geometry& g, const T* x, T* y, cudaStream_t s) {
    g.require_angles();
    ctkb::op_ax<T>(g, x, y, s);
    if (g.comm && g.slab) {
        if (g.band) ctkb::band_reduce<T>(g, y, s);  // partials to the rows' owners
        else ctkb::comm_allreduce(g.comm, y, g.range(), sizeof(T) == 8 ? 1 : 0, s);
    }
}

template <class T>
void atb_dev(ctkb::Geometry& g, int variant, const T* y, T* x, cudaStream_t s) {
    g.require_angles();
    check_variant(variant);
    if (g.band) y = ctkb::band_halo<T>(g, y, s);  // the reached rows other ranks own
    ctkb::op_atb<T>(g, variant, y, x, s);
    if (g.comm && !g.slab) ctkb::comm_allreduce(g.comm, x, g.domain(), sizeof(T) == 8 ? 1 : 0, s);
}

template <class T>
void ax_host(ctkb::Geometry& g, const T* hx, T* hy) {
    const size_t nd = g.domain(), nr = g.range();
    g.host_x.ensure(sizeof(T) * nd);
    g.host_y.ensure(sizeof(T) * nr);
    CTK_CUDA(cudaMemcpyAsync(g.host_x.p, hx, sizeof(T) * nd, cudaMemcpyHostToDevice, g.stream));
    ax_dev<T>(g, g.host_x.as<T>(), g.host_y.as<T>(), g.stream);
    CTK_CUDA(cudaMemcpyAsync(hy, g.host_y.p, sizeof(T) * nr, cudaMemcpyDeviceToHost, g.stream));
    CTK_CUDA(cudaStreamSynchronize(g.stream));
}

template <class T>
void atb_host(ctkb::Geometry& g, int variant, const T* hy, T* hx) {
    const size_t nd = g.domain(), nr = g.range();
    g.host_x.ensure(sizeof(T) * nd);
    g.host_y.ensure(sizeof(T) * nr);
    CTK_CUDA(cudaMemcpyAsync(g.host_y.p, hy, sizeof(T) * nr, cudaMemcpyHostToDevice, g.stream));
    atb_dev<T>(g, variant, g.host_y.as<T>(), g.host_x.as<T>(), g.stream);
    CTK_CUDA(cudaMemcpyAsync(hx, g.host_x.p, sizeof(T) * nd, cudaMemcpyDeviceToHost, g.stream));
    CTK_CUDA(cudaStreamSynchronize(g.stream));
}

template <class T>
void solve_host(ctkb::Geometry& g, int solver, int variant, const T* hb, double lambda, const ctk_hybrid_strategy* st,
                int outer, int inner, int warm, const ctk_solver_opts* o, T* hx, ctk_solve_log* log) {
    if (!hb || !hx) ctkb::fail(CTK_E_PARAMETER, "null host buffer");
    const size_t nd = g.domain(), nr = g.range();
    // the handle's staging buffers (kept between calls, like the solver workspaces)
    ctkb::DevBuf& db = g.host_y;
    ctkb::DevBuf& dx = g.host_x;
    db.ensure(sizeof(T) * nr);
    dx.ensure(sizeof(T) * nd);
    CTK_CUDA(cudaMemcpyAsync(db.p, hb, sizeof(T) * nr, cudaMemcpyHostToDevice, g.stream));
    ctkb::solve_device<T>(g, solver, variant, db.as<T>(), lambda, st, outer, inner, warm, o, dx.as<T>(), log);
    CTK_CUDA(cudaMemcpyAsync(hx, dx.p, sizeof(T) * nd, cudaMemcpyDeviceToHost, g.stream));
    CTK_CUDA(cudaStreamSynchronize(g.stream));
}

ctkb::RedWork global_work() {
    static thread_local ctkb::DevBuf buf;
    buf.ensure(sizeof(double) * (size_t(ctkb::kRedBlocks) * ctkb::kRedSlots + ctkb::kRedSlots));
    ctkb::RedWork w;
    w.partials = buf.as<double>();
    w.results = w.partials + size_t(ctkb::kRedBlocks) * ctkb::kRedSlots;
    return w;
}

template <class T>
void dot_dev(size_t n, const T* x, const T* y, double* out, void* stream) {
    auto s = static_cast<cudaStream_t>(stream);
    auto w = global_work();
    ctkb::reduce_dot<T>(n, x, y, w.results, w, s);
    CTK_CUDA(cudaMemcpyAsync(out, w.results, sizeof(double), cudaMemcpyDeviceToHost, s));
    CTK_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

static void check_vol(int nx, int ny, int nz) {
    if (nx <= 0 || ny <= 0 || nz <= 0) ctkb::fail(CTK_E_DIMENSION, "volume dimensions must be positive");
}

extern "C" {

int ctk_last_error(char* buf, size_t len) {
    if (buf && len) {
        std::strncpy(buf, t_msg.c_str(), len - 1);
        buf[len - 1] = 0;
    }
    return t_code;
}
int ctk_last_error_iteration(void) { return t_iter; }
int ctk_abi_version(void) { return CTK_ABI_VERSION; }

int ctk_geom_create(const ctk_geom_desc* desc, ctk_geom** out) {
    return guard([&] {
        if (!out) ctkb::fail(CTK_E_PARAMETER, "null output handle");
        *out = nullptr;
        *out = reinterpret_cast<ctk_geom*>(ctkb::geometry_create(desc));
    });
}
int ctk_geom_validate(const ctk_geom_desc* desc) {
    return guard([&] { ctkb::geometry_validate(desc); });
}
void ctk_geom_destroy(ctk_geom* g) { delete reinterpret_cast<ctkb::Geometry*>(g); }

int ctk_geom_sizes(const ctk_geom* g, size_t* d, size_t* r) {
    return guard([&] {
        if (d) *d = G(g).domain();
        if (r) *r = G(g).range();
    });
}
int ctk_geom_set_projector(ctk_geom* g, int p) {
    return guard([&] {
        if (p != CTK_PROJ_JOSEPH && p != CTK_PROJ_SIDDON) ctkb::fail(CTK_E_PARAMETER, "unknown projector");
        G(g).projector = p;
    });
}
int ctk_geom_set_slab(ctk_geom* g, int z0, int nz_local) {
    return guard([&] {
        auto& gg = G(g);
        if (nz_local == 0) {
            gg.slab = false;
            gg.z0 = 0;
            gg.nzl = 0;
        } else {
            if (z0 < 0 || nz_local < 1 || z0 + nz_local > gg.nz) ctkb::fail(CTK_E_PARAMETER, "slab outside the volume");
            gg.slab = true;
            gg.z0 = z0;
            gg.nzl = nz_local;
        }
        gg.band = false;  // the row window depends on the slab: ctk_geom_shard_range again
        gg.vx.release();  // padded relayouts depend on the slab height
        gg.vy.release();
    });
}
int ctk_geom_set_bp_partitions(ctk_geom* g, int n) {
    return guard([&] {
        if (n < 1) ctkb::fail(CTK_E_PARAMETER, "partitions must be >= 1");
        G(g).bp_parts = n;
    });
}
int ctk_geom_set_stream(ctk_geom* g, void* stream) {
    return guard([&] {
        auto& gg = G(g);
        if (gg.own_stream && gg.stream) cudaStreamDestroy(gg.stream);
        gg.own_stream = false;
        gg.stream = static_cast<cudaStream_t>(stream);
        if (!stream) {
            CTK_CUDA(cudaStreamCreateWithFlags(&gg.stream, cudaStreamNonBlocking));
            gg.own_stream = true;
        }
    });
}

int ctk_ax_f32(ctk_geom* g, const float* x, float* y, void* s) {
    return guard([&] { ax_dev<float>(G(g), x, y, S(G(g), s)); });
}
int ctk_ax_f64(ctk_geom* g, const double* x, double* y, void* s) {
    return guard([&] { ax_dev<double>(G(g), x, y, S(G(g), s)); });
}
int ctk_atb_f32(ctk_geom* g, int v, const float* y, float* x, void* s) {
    return guard([&] { atb_dev<float>(G(g), v, y, x, S(G(g), s)); });
}
int ctk_atb_f64(ctk_geom* g, int v, const double* y, double* x, void* s) {
    return guard([&] { atb_dev<double>(G(g), v, y, x, S(G(g), s)); });
}
int ctk_ax_pair_f32(ctk_geom* g, const float* x1, float* y1, const float* x2, float* y2, void* s) {
    return guard([&] {
        auto& gg = G(g);
        gg.require_angles();
        if (gg.comm) ctkb::fail(CTK_E_UNSUPPORTED, "ax_pair: not on a sharded handle");
        ctkb::ax2_f32(gg, x1, y1, x2, y2, S(gg, s));
    });
}
int ctk_ax_residual_f32(ctk_geom* g, const float* x, const float* b, double* out, void* s) {
    return guard([&] {
        auto& gg = G(g);
        gg.require_angles();
        if (gg.projector != CTK_PROJ_JOSEPH) ctkb::fail(CTK_E_UNSUPPORTED, "fused residual is Joseph-only");
        auto st = S(gg, s);
        auto w = ctkb::red_work(&gg);
        if (gg.comm && gg.slab) {  // the partial projections must be summed before the difference
            gg.ax_scratch.ensure(gg.range() * sizeof(float));
            ax_dev<float>(gg, x, gg.ax_scratch.as<float>(), st);
            ctkb::reduce_diff_nrm2sq<float>(gg.range(), gg.ax_scratch.as<float>(), b, w.results, w, st);
        } else {
            ctkb::ax_residual_f32(gg, x, b, w.results, st);
        }
        CTK_CUDA(cudaMemcpyAsync(gg.pinned, w.results, sizeof(double), cudaMemcpyDeviceToHost, st));
        CTK_CUDA(cudaStreamSynchronize(st));
        double v = gg.pinned[0];
        if (gg.comm && (!gg.slab || gg.band)) v = ctkb::comm_sum_scalar(gg.comm, v);  // sharded range: partials
        *out = v;
    });
}

int ctk_ax_host_f32(ctk_geom* g, const float* x, float* y) { return guard([&] { ax_host<float>(G(g), x, y); }); }
int ctk_ax_host_f64(ctk_geom* g, const double* x, double* y) { return guard([&] { ax_host<double>(G(g), x, y); }); }
int ctk_atb_host_f32(ctk_geom* g, int v, const float* y, float* x) {
    return guard([&] { atb_host<float>(G(g), v, y, x); });
}
int ctk_atb_host_f64(ctk_geom* g, int v, const double* y, double* x) {
    return guard([&] { atb_host<double>(G(g), v, y, x); });
}

int ctk_dot_f32(size_t n, const float* x, const float* y, double* out, void* s) {
    return guard([&] { dot_dev<float>(n, x, y, out, s); });
}
int ctk_dot_f64(size_t n, const double* x, const double* y, double* out, void* s) {
    return guard([&] { dot_dev<double>(n, x, y, out, s); });
}
int ctk_nrm2_f32(size_t n, const float* x, double* out, void* s) {
    return guard([&] {
        dot_dev<float>(n, x, x, out, s);
        *out = std::sqrt(*out);
    });
}
int ctk_nrm2_f64(size_t n, const double* x, double* out, void* s) {
    return guard([&] {
        dot_dev<double>(n, x, x, out, s);
        *out = std::sqrt(*out);
    });
}
int ctk_axpy_f32(size_t n, double a, const float* x, float* y, void* s) {
    return guard([&] { ctkb::axpy<float>(n, a, x, y, static_cast<cudaStream_t>(s)); });
}
int ctk_axpy_f64(size_t n, double a, const double* x, double* y, void* s) {
    return guard([&] { ctkb::axpy<double>(n, a, x, y, static_cast<cudaStream_t>(s)); });
}
int ctk_scal_f32(size_t n, double a, float* x, void* s) {
    return guard([&] { ctkb::scal<float>(n, a, x, static_cast<cudaStream_t>(s)); });
}
int ctk_scal_f64(size_t n, double a, double* x, void* s) {
    return guard([&] { ctkb::scal<double>(n, a, x, static_cast<cudaStream_t>(s)); });
}

int ctk_make_phantom_f32(int kind, int n, float* out, void* s) {
    return guard([&] {
        if (kind < 0 || kind > 2) ctkb::fail(CTK_E_PARAMETER, "unknown phantom kind");
        if (n < 8) ctkb::fail(CTK_E_PARAMETER, "phantom size must be at least 8");
        ctkb::launch_phantom_f32(kind, n, out, static_cast<cudaStream_t>(s));
    });
}
int ctk_make_phantom_f64(int kind, int n, double* out, void* s) {
    return guard([&] {
        if (kind < 0 || kind > 2) ctkb::fail(CTK_E_PARAMETER, "unknown phantom kind");
        if (n < 8) ctkb::fail(CTK_E_PARAMETER, "phantom size must be at least 8");
        ctkb::launch_phantom_f64(kind, n, out, static_cast<cudaStream_t>(s));
    });
}
int ctk_shepp_logan_3d_f32(int n, float* out, void* s) { return ctk_make_phantom_f32(0, n, out, s); }
int ctk_shepp_logan_3d_f64(int n, double* out, void* s) { return ctk_make_phantom_f64(0, n, out, s); }

#define CTK_STENCIL_API(T, SUF)                                                                                  \
    int ctk_gradient_##SUF(int nx, int ny, int nz, const T* x, T* dx, T* dy, T* dz, void* s) {                \
        return guard([&] {                                                                                   \
            check_vol(nx, ny, nz);                                                                        \
            ctkb::gradient_scaled<T>(nx, ny, nz, x, nullptr, 1.0, dx, dy, dz, static_cast<cudaStream_t>(s)); \
        });                                                                                                  \
    }                                                                                                        \
    int ctk_gradient_adjoint_##SUF(int nx, int ny, int nz, const T* dx, const T* dy, const T* dz, T* out,    \
                                   void* s) {                                                                \
        return guard([&] {                                                                                   \
            check_vol(nx, ny, nz);                                                                        \
            const cudaStream_t st = static_cast<cudaStream_t>(s);                                            \
            CTK_CUDA(cudaMemsetAsync(out, 0, sizeof(T) * size_t(nx) * ny * nz, st));                         \
            ctkb::gradient_adjoint_scaled_add<T>(nx, ny, nz, dx, dy, dz, nullptr, 1.0, out, st);            \
        });                                                                                                  \
    }                                                                                                        \
    int ctk_tv_weights_##SUF(int nx, int ny, int nz, const T* x, double eps, T* w, void* s) {                 \
        return guard([&] {                                                                                   \
            check_vol(nx, ny, nz);                                                                        \
            ctkb::tv_weights<T>(nx, ny, nz, x, eps, w, static_cast<cudaStream_t>(s));                       \
        });                                                                                                  \
    }
CTK_STENCIL_API(float, f32)
CTK_STENCIL_API(double, f64)
#undef CTK_STENCIL_API

int ctk_add_noise_f32(size_t n, const float* in, double i0, double sigma, uint64_t seed, float* out) {
    return guard([&] { ctkb::add_noise<float>(n, in, i0, sigma, seed, out); });
}
int ctk_add_noise_f64(size_t n, const double* in, double i0, double sigma, uint64_t seed, double* out) {
    return guard([&] { ctkb::add_noise<double>(n, in, i0, sigma, seed, out); });
}

#define CTK_SOLVE_HOST(NAME, T, SOLVER)                                                                       \
    int NAME(ctk_geom* g, int variant, const T* b, const ctk_solver_opts* o, T* x, ctk_solve_log* log) {      \
        return guard([&] { solve_host<T>(G(g), SOLVER, variant, b, 0.0, nullptr, 1, 1, 0, o, x, log); });   \
    }
CTK_SOLVE_HOST(ctk_cgls_f32, float, 0)
CTK_SOLVE_HOST(ctk_cgls_f64, double, 0)
CTK_SOLVE_HOST(ctk_lsqr_f32, float, 1)
CTK_SOLVE_HOST(ctk_lsqr_f64, double, 1)
CTK_SOLVE_HOST(ctk_sirt_f32, float, 5)
CTK_SOLVE_HOST(ctk_sirt_f64, double, 5)
CTK_SOLVE_HOST(ctk_ab_gmres_f32, float, 6)
CTK_SOLVE_HOST(ctk_ab_gmres_f64, double, 6)
CTK_SOLVE_HOST(ctk_ba_gmres_f32, float, 7)
CTK_SOLVE_HOST(ctk_ba_gmres_f64, double, 7)
#undef CTK_SOLVE_HOST

int ctk_lsmr_f32(ctk_geom* g, int variant, const float* b, double lambda, const ctk_solver_opts* o, float* x,
                 ctk_solve_log* log) {
    return guard([&] { solve_host<float>(G(g), 2, variant, b, lambda, nullptr, 1, 1, 0, o, x, log); });
}
int ctk_lsmr_f64(ctk_geom* g, int variant, const double* b, double lambda, const ctk_solver_opts* o, double* x,
                 ctk_solve_log* log) {
    return guard([&] { solve_host<double>(G(g), 2, variant, b, lambda, nullptr, 1, 1, 0, o, x, log); });
}
int ctk_hybrid_lsqr_f32(ctk_geom* g, int variant, const float* b, const ctk_hybrid_strategy* s,
                        const ctk_solver_opts* o, float* x, ctk_solve_log* log) {
    return guard([&] { solve_host<float>(G(g), 3, variant, b, 0.0, s, 1, 1, 0, o, x, log); });
}
int ctk_hybrid_lsqr_f64(ctk_geom* g, int variant, const double* b, const ctk_hybrid_strategy* s,
                        const ctk_solver_opts* o, double* x, ctk_solve_log* log) {
    return guard([&] { solve_host<double>(G(g), 3, variant, b, 0.0, s, 1, 1, 0, o, x, log); });
}
int ctk_flsqr_tv_f32(ctk_geom* g, int variant, const float* b, const ctk_hybrid_strategy* s, const ctk_solver_opts* o,
                     float* x, ctk_solve_log* log) {
    return guard([&] { solve_host<float>(G(g), 8, variant, b, 0.0, s, 1, 1, 0, o, x, log); });
}
int ctk_flsqr_tv_f64(ctk_geom* g, int variant, const double* b, const ctk_hybrid_strategy* s,
                     const ctk_solver_opts* o, double* x, ctk_solve_log* log) {
    return guard([&] { solve_host<double>(G(g), 8, variant, b, 0.0, s, 1, 1, 0, o, x, log); });
}
int ctk_cgls_tv_f32(ctk_geom* g, int variant, const float* b, double lambda, int outer, int inner,
                    const ctk_solver_opts* o, int warm, float* x, ctk_solve_log* log) {
    return guard([&] { solve_host<float>(G(g), 4, variant, b, lambda, nullptr, outer, inner, warm, o, x, log); });
}
int ctk_cgls_tv_f64(ctk_geom* g, int variant, const double* b, double lambda, int outer, int inner,
                    const ctk_solver_opts* o, int warm, double* x, ctk_solve_log* log) {
    return guard([&] { solve_host<double>(G(g), 4, variant, b, lambda, nullptr, outer, inner, warm, o, x, log); });
}
int ctk_solve_dev_f32(ctk_geom* g, int solver, int variant, const float* b, double lambda, const ctk_hybrid_strategy* s,
                      int outer, int inner, int warm, const ctk_solver_opts* o, float* x, ctk_solve_log* log) {
    return guard([&] { ctkb::solve_device<float>(G(g), solver, variant, b, lambda, s, outer, inner, warm, o, x, log); });
}
int ctk_solve_dev_f64(ctk_geom* g, int solver, int variant, const double* b, double lambda,
                      const ctk_hybrid_strategy* s, int outer, int inner, int warm, const ctk_solver_opts* o, double* x,
                      ctk_solve_log* log) {
    return guard([&] { ctkb::solve_device<double>(G(g), solver, variant, b, lambda, s, outer, inner, warm, o, x, log); });
}

int ctk_projected_gcv_lambda(const double* H, int k, double beta1, double* out) {
    return guard([&] {
        if (!H || !out || k < 1) ctkb::fail(CTK_E_PARAMETER, "projected problem must have a (k+1) x k matrix, k >= 1");
        *out = ctkb::gcv_lambda(std::vector<double>(H, H + size_t(k + 1) * k), k, beta1);
    });
}
int ctk_projected_dp_lambda(const double* H, int k, double beta1, double nl, double* out) {
    return guard([&] {
        if (!H || !out || k < 1) ctkb::fail(CTK_E_PARAMETER, "projected problem must have a (k+1) x k matrix, k >= 1");
        *out = ctkb::dp_lambda(std::vector<double>(H, H + size_t(k + 1) * k), k, beta1, nl);
    });
}
int ctk_projected_tikhonov(const double* H, int k, double beta1, double lambda, double* y, double* fit) {
    return guard([&] {
        if (!H || !y || k < 1) ctkb::fail(CTK_E_PARAMETER, "projected problem must have a (k+1) x k matrix, k >= 1");
        auto v = ctkb::projected_tikhonov(std::vector<double>(H, H + size_t(k + 1) * k), k, beta1, lambda, fit);
        std::copy(v.begin(), v.end(), y);
    });
}

int ctk_shard_slabs(int nz, int nranks, int rank, int* z0, int* count) {
    return ctk_shard_angles(nz, nranks, rank, z0, count);  // the same contiguous block partition
}
int ctk_shard_angles(int n_angles, int nranks, int rank, int* first, int* count) {
    return guard([&] {
        if (n_angles < 1 || nranks < 1 || rank < 0 || rank >= nranks) ctkb::fail(CTK_E_PARAMETER, "invalid sharding");
        // contiguous blocks; the first (n_angles % nranks) ranks take one extra angle
        const int base = n_angles / nranks, extra = n_angles % nranks;
        *first = rank * base + std::min(rank, extra);
        *count = base + (rank < extra ? 1 : 0);
    });
}
int ctk_comm_create(const ctk_comm_callbacks* cb, ctk_comm** out) {
    return guard([&] {
        if (!cb || !out) ctkb::fail(CTK_E_PARAMETER, "null callbacks");
        if (cb->nranks < 1 || cb->rank < 0 || cb->rank >= cb->nranks) ctkb::fail(CTK_E_PARAMETER, "invalid rank / nranks");
        auto* c = new ctkb::Comm();
        c->cb = *cb;
        *out = reinterpret_cast<ctk_comm*>(c);
    });
}
int ctk_nccl_get_unique_id(void* out128) { return guard([&] { ctkb::nccl_unique_id(out128); }); }
int ctk_comm_adopt_nccl(void* nccl_comm, int nranks, int rank, ctk_comm** out) {
    return guard([&] { *out = reinterpret_cast<ctk_comm*>(ctkb::comm_adopt_nccl(nccl_comm, nranks, rank)); });
}
int ctk_comm_create_nccl(const void* id, int nranks, int rank, ctk_comm** out) {
    return guard([&] { *out = reinterpret_cast<ctk_comm*>(ctkb::comm_create_nccl(id, nranks, rank)); });
}
void ctk_comm_destroy(ctk_comm* c) { ctkb::comm_destroy(reinterpret_cast<ctkb::Comm*>(c)); }
int ctk_geom_attach_comm(ctk_geom* g, ctk_comm* c) {
    return guard([&] {
        G(g).comm = reinterpret_cast<ctkb::Comm*>(c);
        G(g).band = false;
    });
}

int ctk_geom_shard_range(ctk_geom* g) {
    return guard([&] {
        auto& gg = G(g);
        if (!gg.slab || !gg.comm) ctkb::fail(CTK_E_PARAMETER, "band-sharded range needs a slab and a communicator");
        const int R = gg.comm->cb.nranks, me = gg.comm->cb.rank;
        const std::vector<double> z0s = ctkb::comm_allgather_scalar(gg.comm, double(gg.z0));
        const std::vector<double> nzs = ctkb::comm_allgather_scalar(gg.comm, double(gg.nzl));
        std::vector<int> z0i(static_cast<size_t>(R)), nzi(static_cast<size_t>(R));
        for (int r = 0; r < R; ++r) {
            z0i[size_t(r)] = int(z0s[size_t(r)]);
            nzi[size_t(r)] = int(nzs[size_t(r)]);
        }
        gg.bt0.assign(size_t(R), 0);
        gg.bt1.assign(size_t(R), 0);
        gg.bo0.assign(size_t(R), 0);
        gg.bo1.assign(size_t(R), 0);
        ctkb::band_partition(gg.mode, gg.nx, gg.ny, gg.nz, gg.nv, gg.h, gg.du, gg.dso, gg.dod, R, z0i.data(),
                             nzi.data(), gg.bt0.data(), gg.bt1.data(), gg.bo0.data(), gg.bo1.data());
        const size_t m = size_t(me);
        const int t0 = gg.bt0[m], t1 = std::max(gg.bt1[m], gg.bt0[m]), o0 = gg.bo0[m], o1 = gg.bo1[m];
        gg.w0 = t1 > t0 ? std::min(t0, o0) : o0;
        gg.nw = std::max(std::max(t1, o1), gg.w0 + 1) - gg.w0;
        gg.band = true;
    });
}

int ctk_geom_range_rows(const ctk_geom* g, int* w0, int* nw, int* o0, int* no) {
    return guard([&] {
        auto& gg = G(g);
        const int me = gg.band ? gg.comm->cb.rank : 0;
        if (w0) *w0 = gg.band ? gg.w0 : 0;
        if (nw) *nw = gg.band ? gg.nw : gg.nv;
        if (o0) *o0 = gg.band ? gg.bo0[size_t(me)] : 0;
        if (no) *no = gg.band ? gg.bo1[size_t(me)] - gg.bo0[size_t(me)] : gg.nv;
    });
}

int ctk_band_partition(const ctk_geom_desc* d, int nranks, const int* z0s, const int* nzs, int* t0, int* t1, int* o0,
                       int* o1) {
    return guard([&] {
        ctkb::geometry_validate(d);
        if (!z0s || !nzs || !t0 || !t1 || !o0 || !o1) ctkb::fail(CTK_E_PARAMETER, "null partition array");
        ctkb::band_partition(d->mode, d->nx, d->ny, d->nz, d->nv, d->spacing, d->detector_pixel_size,
                             d->source_to_origin, d->origin_to_detector, nranks, z0s, nzs, t0, t1, o0, o1);
    });
}

uint64_t ctk_launch_count(void) { return ctkb::launch_count(); }
double ctk_geom_last_kernel_ms(ctk_geom* g) {
    float ms = -1.f;
    guard([&] {
        auto& gg = G(g);
        CTK_CUDA(cudaEventSynchronize(gg.ev1));
        CTK_CUDA(cudaEventElapsedTime(&ms, gg.ev0, gg.ev1));
    });
    return double(ms);
}

}  // extern "C"
