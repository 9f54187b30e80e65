/*
 * ctk_b200.h -- C-ABI of the B200-native Ax / A^T b hot path of ctkrylov
 * (arXiv 2211.14212).  Plain pointers and sizes only; no torch or C++ types.
 *
 * The reference has no C-ABI (its FFI is an empty pybind11 `_core`,
 * bindings/bindings.cpp:1-2); every entry point below replaces a C++ interface of the
 * reference, cited per declaration as `file:line` under /root/reference/proj.
 * INTEGRATION.md shows the ctypes / pybind11 / C++ bindings a maintainer would add.
 *
 * Layouts (identical to the reference):
 *   domain (volume)      x[i + nx*(j + ny*k)]                 types.hpp:50-70
 *   range  (projections) y[iu + nu*(iv + nv*a)]               types.hpp:80-102
 * Ownership: callers own every buffer; outputs are overwritten entirely
 * (operators.hpp:102-113).  One in-flight call per ctk_geom; distinct handles may be
 * used concurrently from different threads.
 *
 * Precision: *_f32 entry points run the sm_100a performance kernels (fp32 data,
 * fp64 per-ray setup, fp64 reductions); *_f64 entry points run the exact-parity
 * kernels, which reproduce the reference's IEEE operation sequence for T=double.
 */
#ifndef CTK_B200_H
#define CTK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 2: ctk_comm_callbacks gained the `exchange` member (band-sharded range, p2p halos) -- callers
 * must zero-initialise it when they do not provide one. */
#define CTK_ABI_VERSION 2

/* Error taxonomy of types.hpp:14-31 (DimensionError, GeometryError, ParameterError,
 * DegenerateInputError, NumericalError) plus device failures. */
typedef enum {
    CTK_OK = 0,
    CTK_E_DIMENSION = 1,
    CTK_E_GEOMETRY = 2,
    CTK_E_PARAMETER = 3,
    CTK_E_DEGENERATE = 4,
    CTK_E_NUMERICAL = 5,
    CTK_E_CUDA = 6,
    CTK_E_UNSUPPORTED = 7
} ctk_status;

/* BeamMode, geometry.hpp:11 */
typedef enum { CTK_PARALLEL2D = 0, CTK_PARALLEL3D = 1, CTK_CONE3D = 2 } ctk_beam_mode;
/* BackprojectVariant, projector.hpp:16 */
typedef enum { CTK_BP_MATCHED = 0, CTK_BP_VOXEL_DRIVEN = 1 } ctk_bp_variant;
/* Forward model. Joseph = projector.hpp:48-122; Siddon is new. */
typedef enum { CTK_PROJ_JOSEPH = 0, CTK_PROJ_SIDDON = 1 } ctk_projector;
/* StopReason, solve_log.hpp:16 */
typedef enum { CTK_STOP_MAX_ITERS = 0, CTK_STOP_RESIDUAL_INCREASE = 1, CTK_STOP_TOLERANCE = 2, CTK_STOP_BREAKDOWN = 3 } ctk_stop_reason;
/* LambdaStrategy, hybrid.hpp:13 */
typedef enum { CTK_LAMBDA_FIXED = 0, CTK_LAMBDA_DP = 1, CTK_LAMBDA_GCV = 2 } ctk_lambda_strategy;

/* ConeGeometry, geometry.hpp:24-33 (+ VolumeShape, types.hpp:35-41). */
typedef struct {
    int mode;                   /* ctk_beam_mode */
    double source_to_origin;    /* mm, cone3d only */
    double origin_to_detector;  /* mm */
    double detector_pixel_size; /* mm */
    int nu, nv;
    int nx, ny, nz;
    double spacing;             /* mm per voxel */
    int n_angles;
    const double* angles;       /* radians; reduced by canonical_angle (types.hpp:172-177) */
} ctk_geom_desc;

typedef struct ctk_geom ctk_geom;
typedef struct ctk_comm ctk_comm;

/* ---- errors ---------------------------------------------------------------------- */
/* Thread-local message of the last failing call on this thread; returns its status. */
int ctk_last_error(char* buf, size_t len);
/* Iteration carried by the last CTK_E_NUMERICAL (NumericalError::iteration, types.hpp:27-31). */
int ctk_last_error_iteration(void);
int ctk_abi_version(void);

/* ---- geometry (replaces ConeGeometry::validate + projector_pair capture,
 *      geometry.hpp:35-54, operators.hpp:91-101) -------------------------------------- */
int ctk_geom_create(const ctk_geom_desc* desc, ctk_geom** out);
/* ConeGeometry::validate alone (geometry.hpp:35-54): same checks, order and messages as
 * ctk_geom_create, no device work (host-side validation for bindings). */
int ctk_geom_validate(const ctk_geom_desc* desc);
void ctk_geom_destroy(ctk_geom* g);
/* domain_size = nx*ny*nz, range_size = n_angles*nu*nv (operators.hpp:98-99) */
int ctk_geom_sizes(const ctk_geom* g, size_t* domain_size, size_t* range_size);
/* Forward model used by ctk_ax_* / matched ctk_atb_* (default Joseph). */
int ctk_geom_set_projector(ctk_geom* g, int projector);
/* Partition count used by the exact f64 matched A^T b to reproduce the reference's
 * OpenMP summation order (projector.hpp:172-201): min(OMP threads, n_angles). Default 1. */
int ctk_geom_set_bp_partitions(ctk_geom* g, int nparts);
/* Stream for solver / host-pointer calls (cudaStream_t; NULL = the handle's own stream). */
int ctk_geom_set_stream(ctk_geom* g, void* stream);

/* ---- operators on DEVICE pointers (forward_project, projector.hpp:134-162;
 *      back_project, projector.hpp:283-297).  Asynchronous on `stream` (a cudaStream_t;
 *      NULL = the legacy default stream, as everywhere in CUDA). ----------------------- */
int ctk_ax_f32(ctk_geom* g, const float* d_x, float* d_y, void* stream);
int ctk_ax_f64(ctk_geom* g, const double* d_x, double* d_y, void* stream);
int ctk_atb_f32(ctk_geom* g, int variant, const float* d_y, float* d_x, void* stream);
int ctk_atb_f64(ctk_geom* g, int variant, const double* d_y, double* d_x, void* stream);
/* Fused explicit residual: out = ||A x - b||^2 (fp64), y never stored (solve_log.hpp:111-115). */
int ctk_ax_residual_f32(ctk_geom* g, const float* d_x, const float* d_b, double* h_out, void* stream);
/* Two forward projections in one ray march: d_y1 = A d_x1, d_y2 = A d_x2 (f32, Joseph or Siddon, on a
 * whole-volume handle; CTK_E_UNSUPPORTED otherwise).  No reference counterpart: the solvers
 * use it for the explicit residual's A x (solve_log.hpp:111-115) together with the next
 * Krylov A v.  Each output is bit-identical to ctk_ax_f32's. */
int ctk_ax_pair_f32(ctk_geom* g, const float* d_x1, float* d_y1, const float* d_x2, float* d_y2, void* stream);

/* ---- operators on HOST pointers: OperatorPair::forward / back semantics
 *      (operators.hpp:18-45, 102-113).  Synchronous. ---------------------------------- */
int ctk_ax_host_f32(ctk_geom* g, const float* h_x, float* h_y);
int ctk_ax_host_f64(ctk_geom* g, const double* h_x, double* h_y);
int ctk_atb_host_f32(ctk_geom* g, int variant, const float* h_y, float* h_x);
int ctk_atb_host_f64(ctk_geom* g, int variant, const double* h_y, double* h_x);

/* ---- BLAS-1 (types.hpp:136-158) on device pointers; fp64 accumulation in a fixed
 *      reduction order (run-to-run bitwise deterministic).  Results to host. ---------- */
int ctk_dot_f32(size_t n, const float* d_x, const float* d_y, double* h_out, void* stream);
int ctk_dot_f64(size_t n, const double* d_x, const double* d_y, double* h_out, void* stream);
int ctk_nrm2_f32(size_t n, const float* d_x, double* h_out, void* stream);
int ctk_nrm2_f64(size_t n, const double* d_x, double* h_out, void* stream);
int ctk_axpy_f32(size_t n, double alpha, const float* d_x, float* d_y, void* stream);
int ctk_axpy_f64(size_t n, double alpha, const double* d_x, double* d_y, void* stream);
int ctk_scal_f32(size_t n, double alpha, float* d_x, void* stream);
int ctk_scal_f64(size_t n, double alpha, double* d_x, void* stream);

/* ---- synthetic input: make_phantom (phantom.hpp:118-145) rasterised on the device -----
 * kind follows PhantomKind (phantom.hpp:13): 0 shepp_logan_3d (n^3), 1 shepp_logan_2d
 * (n*n*1), 2 piecewise_blocks (n*n*1).  Bit-identical to the reference's make_phantom<T>. */
#define CTK_PHANTOM_SHEPP_LOGAN_3D 0
#define CTK_PHANTOM_SHEPP_LOGAN_2D 1
#define CTK_PHANTOM_PIECEWISE_BLOCKS 2
int ctk_make_phantom_f32(int kind, int n, float* d_out, void* stream);
int ctk_make_phantom_f64(int kind, int n, double* d_out, void* stream);
int ctk_shepp_logan_3d_f32(int n, float* d_out, void* stream); /* = make_phantom(0, n) */
int ctk_shepp_logan_3d_f64(int n, double* d_out, void* stream);

/* ---- forward-difference gradient and its adjoint (gradient.hpp:9-54), IRN TV weights
 * (tv.hpp:17-43), on device pointers of an nx*ny*nz volume (x fastest).  The gradient and
 * its adjoint are bit-identical to the reference's loops; the weights agree to an ulp (the
 * device pow).  ctk_tv_weights takes eps (tv_epsilon: 1e-4 max|x|, > 0); the reference's
 * all-ones case for eps == 0 is the caller's.  ctk_gradient_adjoint overwrites out. */
int ctk_gradient_f32(int nx, int ny, int nz, const float* d_x, float* d_dx, float* d_dy, float* d_dz, void* stream);
int ctk_gradient_f64(int nx, int ny, int nz, const double* d_x, double* d_dx, double* d_dy, double* d_dz, void* stream);
int ctk_gradient_adjoint_f32(int nx, int ny, int nz, const float* d_dx, const float* d_dy, const float* d_dz,
                             float* d_out, void* stream);
int ctk_gradient_adjoint_f64(int nx, int ny, int nz, const double* d_dx, const double* d_dy, const double* d_dz,
                             double* d_out, void* stream);
int ctk_tv_weights_f32(int nx, int ny, int nz, const float* d_x, double eps, float* d_w, void* stream);
int ctk_tv_weights_f64(int nx, int ny, int nz, const double* d_x, double eps, double* d_w, void* stream);

/* ---- count-domain noise, add_noise (noise.hpp:26-47) on HOST buffers ----------------
 * One mt19937_64 stream walked in detector-index order (a Poisson then a Gaussian draw
 * per sample, libstdc++ distributions): sequential by definition, so it stays on the
 * host and is bit-identical to the reference built with the
 * same C++ standard library.  in/out may alias.  Errors: PARAMETER (i0 <= 0, sigma < 0),
 * DEGENERATE (a negative line integral, checked before any output is written). */
int ctk_add_noise_f32(size_t n, const float* h_in, double i0, double sigma, uint64_t seed, float* h_out);
int ctk_add_noise_f64(size_t n, const double* h_in, double i0, double sigma, uint64_t seed, double* h_out);

/* ---- solvers (solvers.hpp:13-231, hybrid.hpp:76-116, tv.hpp:45-110) ---------------- */
/* SolverOptions, solve_log.hpp:42-57 */
typedef struct {
    int max_iters;
    int stop_on_explicit_residual_increase;
    double residual_tolerance;
    int reorth;
    const void* ground_truth; /* HOST pointer of T (f32/f64 per entry point) or NULL */
    /* iterate_observer test hook (solve_log.hpp:50-51): called with a HOST copy of x_k */
    void (*iterate_observer)(int k, const void* h_x, size_t n, void* user);
    void* observer_user;
} ctk_solver_opts;

/* SolveResult + ConvergenceLog, solve_log.hpp:28-76.  Arrays are caller-allocated with
 * `capacity` entries (max_iters, or outer*inner for cgls_tv). */
typedef struct {
    int capacity;
    double* implicit_residual;
    double* explicit_residual;
    double* relative_error;
    double* lambda;
    int* outer_starts;  /* cgls_tv; capacity >= outer iterations */
    int iterations;     /* entries written to implicit/explicit */
    int n_relative_error;
    int n_lambda;
    int n_outer_starts;
    int iterations_run;
    int stop_reason;    /* ctk_stop_reason */
    int stored_domain_basis;
    int stored_range_basis;
    /* SolveResult::warnings (solve_log.hpp:69): flsqr_tv records the iterations whose inner
     * CG did not converge ("tv preconditioner: inner CG not converged at iteration k",
     * tv.hpp:170-172).  Caller-allocated, `capacity` entries, may be NULL. */
    int* warning_iterations;
    int n_warnings;
} ctk_solve_log;

/* HybridStrategy, hybrid.hpp:15-33 */
typedef struct {
    int kind;            /* ctk_lambda_strategy */
    double lambda;       /* fixed */
    double noise_level;  /* dp */
} ctk_hybrid_strategy;

/* Host-pointer solvers (the reference's signatures: pair = (geom, variant)). */
int ctk_cgls_f32(ctk_geom* g, int variant, const float* h_b, const ctk_solver_opts* o, float* h_x, ctk_solve_log* log);
int ctk_cgls_f64(ctk_geom* g, int variant, const double* h_b, const ctk_solver_opts* o, double* h_x, ctk_solve_log* log);
int ctk_lsqr_f32(ctk_geom* g, int variant, const float* h_b, const ctk_solver_opts* o, float* h_x, ctk_solve_log* log);
int ctk_lsqr_f64(ctk_geom* g, int variant, const double* h_b, const ctk_solver_opts* o, double* h_x, ctk_solve_log* log);
int ctk_lsmr_f32(ctk_geom* g, int variant, const float* h_b, double lambda, const ctk_solver_opts* o, float* h_x, ctk_solve_log* log);
int ctk_lsmr_f64(ctk_geom* g, int variant, const double* h_b, double lambda, const ctk_solver_opts* o, double* h_x, ctk_solve_log* log);
int ctk_hybrid_lsqr_f32(ctk_geom* g, int variant, const float* h_b, const ctk_hybrid_strategy* s, const ctk_solver_opts* o, float* h_x, ctk_solve_log* log);
int ctk_hybrid_lsqr_f64(ctk_geom* g, int variant, const double* h_b, const ctk_hybrid_strategy* s, const ctk_solver_opts* o, double* h_x, ctk_solve_log* log);
int ctk_cgls_tv_f32(ctk_geom* g, int variant, const float* h_b, double lambda, int outer_iters, int inner_iters, const ctk_solver_opts* o, int warm_start, float* h_x, ctk_solve_log* log);
int ctk_cgls_tv_f64(ctk_geom* g, int variant, const double* h_b, double lambda, int outer_iters, int inner_iters, const ctk_solver_opts* o, int warm_start, double* h_x, ctk_solve_log* log);
/* SIRT (solvers.hpp:233-287) and AB/BA-GMRES (gmres.hpp:101-114): same signature as cgls. */
int ctk_sirt_f32(ctk_geom* g, int variant, const float* h_b, const ctk_solver_opts* o, float* h_x, ctk_solve_log* log);
int ctk_sirt_f64(ctk_geom* g, int variant, const double* h_b, const ctk_solver_opts* o, double* h_x, ctk_solve_log* log);
int ctk_ab_gmres_f32(ctk_geom* g, int variant, const float* h_b, const ctk_solver_opts* o, float* h_x, ctk_solve_log* log);
int ctk_ab_gmres_f64(ctk_geom* g, int variant, const double* h_b, const ctk_solver_opts* o, double* h_x, ctk_solve_log* log);
int ctk_ba_gmres_f32(ctk_geom* g, int variant, const float* h_b, const ctk_solver_opts* o, float* h_x, ctk_solve_log* log);
int ctk_ba_gmres_f64(ctk_geom* g, int variant, const double* h_b, const ctk_solver_opts* o, double* h_x, ctk_solve_log* log);
/* flsqr_tv (tv.hpp:177-185): flexible hybrid LSQR with the TV priorconditioner; the
 * strategy must be fixed or gcv (dp -> CTK_E_PARAMETER, as in hybrid.hpp:135-136). */
int ctk_flsqr_tv_f32(ctk_geom* g, int variant, const float* h_b, const ctk_hybrid_strategy* s, const ctk_solver_opts* o, float* h_x, ctk_solve_log* log);
int ctk_flsqr_tv_f64(ctk_geom* g, int variant, const double* h_b, const ctk_hybrid_strategy* s, const ctk_solver_opts* o, double* h_x, ctk_solve_log* log);

/* Device-resident variants: b and x are DEVICE pointers; identical semantics.
 * solver: 0 cgls, 1 lsqr, 2 lsmr, 3 hybrid_lsqr, 4 cgls_tv, 5 sirt, 6 ab_gmres,
 * 7 ba_gmres, 8 flsqr_tv (reads `s`).  `lambda` is the LSMR
 * damping / TV weight; hybrid reads `s`; cgls_tv reads outer/inner/warm_start. */
int ctk_solve_dev_f32(ctk_geom* g, int solver, int variant, const float* d_b, double lambda,
                      const ctk_hybrid_strategy* s, int outer_iters, int inner_iters, int warm_start,
                      const ctk_solver_opts* o, float* d_x, ctk_solve_log* log);
int ctk_solve_dev_f64(ctk_geom* g, int solver, int variant, const double* d_b, double lambda,
                      const ctk_hybrid_strategy* s, int outer_iters, int inner_iters, int warm_start,
                      const ctk_solver_opts* o, double* d_x, ctk_solve_log* log);

/* ---- host fp64 projected-problem helpers of hybrid LSQR (no GPU needed).  H is the
 *      (k+1) x k projected matrix, row-major. ------------------------------------------- */
/* gcv_lambda, regparam.hpp:114-159 (returns the linear-convention parameter) */
int ctk_projected_gcv_lambda(const double* H, int k, double beta1, double* out);
/* dp_lambda, regparam.hpp:79-113 */
int ctk_projected_dp_lambda(const double* H, int k, double beta1, double noise_level, double* out);
/* projected_tikhonov, hybrid.hpp:37-55: y (k entries) and the data-fit residual */
int ctk_projected_tikhonov(const double* H, int k, double beta1, double lambda, double* y, double* fit_resid);

/* ---- multi-GPU angle sharding ------------------------------------- */
/* Contiguous angle block of rank r among G ranks: [first, first+count). */
int ctk_shard_angles(int n_angles, int nranks, int rank, int* first, int* count);
/* Collectives as callbacks (NCCL below, or any transport e.g. torch.distributed).
 * allreduce_sum: in-place sum of `count` elements (dtype 0=f32, 1=f64) of a DEVICE buffer
 * on `stream`; allgather_f64: gathers one host double per rank into out[nranks]. */
/* One point-to-point transfer of an exchange: send or receive `count` elements of a DEVICE
 * buffer to / from rank `peer`. */
typedef struct {
    int peer;
    int is_send;
    void* d_buf;
    size_t count;
} ctk_p2p_op;
typedef struct {
    int rank, nranks;
    int (*allreduce_sum)(void* d_buf, size_t count, int dtype, void* stream, void* user);
    int (*allgather_f64)(double value, double* h_out, void* user);
    void* user;
    /* exchange (optional; needed by the band-sharded range, ctk_geom_shard_range): run all
     * n_ops transfers (dtype 0=f32, 1=f64), ordered on `stream` after the kernels queued
     * before and before the ones queued after; NULL in older callers. */
    int (*exchange)(const ctk_p2p_op* ops, int n_ops, int dtype, void* stream, void* user);
} ctk_comm_callbacks;
int ctk_comm_create(const ctk_comm_callbacks* cb, ctk_comm** out);
/* NCCL (dlopen'd libnccl.so.2): unique id is 128 bytes, exchanged by the caller. */
int ctk_nccl_get_unique_id(void* out128);
int ctk_comm_create_nccl(const void* id128, int nranks, int rank, ctk_comm** out);
/* Adopt a communicator the caller already initialised (an ncclComm_t passed as void*, e.g.
 * the one behind a torch.distributed NCCL process group).  The caller keeps ownership:
 * ctk_comm_destroy does not destroy it, and it must outlive the ctk_comm. */
int ctk_comm_adopt_nccl(void* nccl_comm, int nranks, int rank, ctk_comm** out);
void ctk_comm_destroy(ctk_comm* c);
/* Attach a communicator.  Angle sharding (no slab set): the handle's angles are this
 * rank's shard; A^T b partial volumes are sum-reduced and range-space dots are summed over
 * ranks in rank order.  z-slab sharding (ctk_geom_set_slab): domain vectors are this
 * rank's slab; A x partial projections are sum-reduced, domain-space dots are summed in
 * rank order and the TV stencils exchange one-slice halos. */
int ctk_geom_attach_comm(ctk_geom* g, ctk_comm* c);

/* ---- z-slab sharding --------------------------------------- */
/* Contiguous z-slab of rank r among G ranks: slices [z0, z0+count). */
int ctk_shard_slabs(int nz, int nranks, int rank, int* z0, int* count);
/* The handle's domain vectors hold slices [z0, z0+nz_local) of the geometry's nz (the
 * geometry, angles and detector stay global); nz_local = 0 restores the whole volume.
 * Implemented for the f32 Joseph operators (others return CTK_E_UNSUPPORTED at apply). */
int ctk_geom_set_slab(ctk_geom* g, int z0, int nz_local);
/* Band-sharded range (needs a slab and an attached communicator whose ranks hold the slabs
 * of ctk_shard_slabs in rank order): range vectors then hold only the detector rows
 * [w0, w0 + nw) of every view -- the rows this slab's rays reach plus the rows this rank
 * owns, [o0, o0 + no); rows held but not owned are kept at zero.  A x partials are summed by
 * the rows' owners (point-to-point, rank order) and A^T b fetches the reached rows it does
 * not own from their owners; per-rank memory O(N_vox / G + band).  Collective: every rank
 * calls it.  ctk_geom_sizes then reports the local range size n_angles * nw * nu. */
int ctk_geom_shard_range(ctk_geom* g);
int ctk_geom_range_rows(const ctk_geom* g, int* w0, int* nw, int* o0, int* no);
/* The partition itself, host only: slabs [z0s[r], z0s[r] + nzs[r]) tiling nz in rank order
 * -> reached rows [t0[r], t1[r]) and owned rows [o0[r], o1[r]) (a partition of [0, nv)). */
int ctk_band_partition(const ctk_geom_desc* desc, int nranks, const int* z0s, const int* nzs, int* t0, int* t1,
                       int* o0, int* o1);

/* ---- instrumentation ----------------------------------------------------------------- */
/* Number of this library's kernel launches since load (for bench gpu_launches). */
uint64_t ctk_launch_count(void);
/* Device time of the last ctk_ax_* / ctk_atb_* main kernel on this handle (CUDA events
 * recorded on its stream around that kernel), ms.  Synchronises the handle's last event. */
double ctk_geom_last_kernel_ms(ctk_geom* g);

#ifdef __cplusplus
}
#endif
#endif /* CTK_B200_H */
