// Internal declarations of libctk_b200.so (not part of the C-ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ctk_b200.h"

namespace ctkb {

// ---- errors: C++ exceptions inside, status codes at the C-ABI -------------------------
struct Error : std::runtime_error {
    int code;
    int iteration;
    Error(int c, const std::string& m, int it = 0) : std::runtime_error(m), code(c), iteration(it) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg, int it = 0) { throw Error(code, msg, it); }

#define CTK_CUDA(call)                                                                          \
    do {                                                                                        \
        cudaError_t e_ = (call);                                                                \
        if (e_ != cudaSuccess)                                                                  \
            ::ctkb::fail(CTK_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));       \
    } while (0)

// Checks the launch that was just issued and counts it (ctk_launch_count).
void after_launch(const char* what);

// ---- device buffers --------------------------------------------------------------------
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf();
    // grows (never shrinks); returns true when (re)allocated, contents then undefined
    bool ensure(size_t nbytes);
    void release();
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

// ---- kernel-side geometry (passed by value) --------------------------------------------
struct KGeom {
    int mode, nu, nv, nx, ny, nz, na;
    int nzg, z0;                  // z-slab: the handle holds slices [z0, z0 + nz) of nzg
    int w0, nw;                   // range rows held: [w0, w0 + nw) of nv (band-sharded range; else 0, nv)
    int has_zrays;
    double dso, dod, du, h;
    const double2* ctst;          // per view (cos, sin), host libm values
    const float4* col;            // per (view, iu): fh0, fhd, g0, gd   (f32 separable model)
    const double4* col64;         // the same in fp64 (anchors of the f32 positions, f32_common.cuh)
    const unsigned char* colaxis; // per (view, iu): 0 = x-dominant, 1 = y-dominant
    const double2* colstep;       // per (view, iu): (dx^2+dy^2, |d_A|) of the unnormalised ray
    const int4* vclass;           // per view: column hull [x.. y] of x-dominant, [z.. w] of y-dominant columns
#ifdef CTK_CHECKED
    unsigned* chk;                // checked builds: bounds-violation bits
#endif
    // (KGeom is kept at 128 bytes in the product build: one more word measured +12 % on the
    // plane backprojector -- its register allocation spills more beyond that size)
};

// ---- the geometry handle ---------------------------------------------------------------
struct Comm;

struct Geometry {
    int mode = 0, nu = 0, nv = 0, nx = 0, ny = 0, nz = 0, na = 0;
    double dso = 0, dod = 0, du = 0, h = 0;
    std::vector<double> angles;  // canonical
    std::vector<double> ct, st;
    bool angles_valid = true;    // ProjectionSet::validate (types.hpp:104-117), raised at apply time
    std::string angles_msg;
    bool has_zrays = false;      // any cone ray with |d_z| dominant
    int projector = CTK_PROJ_JOSEPH;
    int bp_parts = 1;
    // z-slab sharding: domain vectors hold slices [z0, z0 + nzl) of nz
    bool slab = false;
    int z0 = 0, nzl = 0;
    // band-sharded range (ctk_geom_shard_range, z-slab + communicator): range vectors hold
    // detector rows [w0, w0 + nw) of every view -- the rows this slab's rays reach (t0..t1)
    // and the rows this rank owns (o0..o1); per rank r of the communicator bt0/bt1 (reached)
    // and bo0/bo1 (owned, a partition of [0, nv)) -- SURVEY.md 8(e)
    bool band = false;
    int w0 = 0, nw = 0;
    std::vector<int> bt0, bt1, bo0, bo1;
    DevBuf band_send, band_recv, band_scratch;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    Comm* comm = nullptr;

    // device tables
    DevBuf d_ctst, d_col, d_col64, d_colaxis, d_colstep;
    DevBuf d_vorder;  // views grouped by ray class (x-dominant first) for L2 reuse in Ax
    DevBuf d_vclass;  // per view: hull of the columns of each ray class (matched A^T b batching)
    DevBuf d_chk;     // checked builds: one word of bounds-violation bits (kernels atomicOr into it)
    DevBuf d_rayinv;  // per ray: 1/d of make_ray, for the exact gathers (built on first use)
    DevBuf bp_parts_buf;  // view-chunk partial volumes of the plane A^T b (small problems)
    bool rayinv_ready = false;
    DevBuf d_walk;    // per ray: the plan_walk parameters of the exact f64 path (built on first use)
    DevBuf d_vscale;  // per view: parallel-beam scale of the voxel-driven f64 path (built on first use)
    bool vscale_ready = false;
    bool walk_ready = false;
    // workspaces (grown lazily)
    DevBuf vx, vy;      // padded f32 relayouts for x- / y-dominant rays
    DevBuf vx2, vy2;    // the same layouts with two volumes interleaved (float2), for ax2_f32
    DevBuf dx64, dy64;  // z-fast f64 copies for the exact forward: X[i][j][k], Y[j][i][k]
    DevBuf proj_t;      // transposed (and step-scaled) projections for the gathers
    DevBuf host_x, host_y;  // device staging for host-pointer entry points
    DevBuf ax_scratch;      // A x of the chunked explicit residual
    DevBuf red;         // reduction scratch (partials + results)
    double* pinned = nullptr;  // host-side reduction results
    // solver workspaces, kept across solves on this handle (cudaMalloc/cudaFree per solve
    // cost several ms and synchronise); slots are handed out in call order and only grow
    std::vector<std::unique_ptr<DevBuf>> ws_pool;
    size_t ws_next = 0;
    DevBuf& ws_take() {
        if (ws_next == ws_pool.size()) ws_pool.emplace_back(new DevBuf());
        return *ws_pool[ws_next++];
    }
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;

    size_t domain() const { return size_t(nx) * ny * (slab ? nzl : nz); }
    int nz_local() const { return slab ? nzl : nz; }
    size_t range() const { return size_t(na) * nu * (band ? nw : nv); }
    int rows_local() const { return band ? nw : nv; }
    KGeom kgeom() const;
    void require_angles() const;
    ~Geometry();
};

// ---- kernels (launch wrappers) ---------------------------------------------------------
// exact f64 path (kernels_f64.cu, compiled with --fmad=false)
void launch_ax_exact_f64(Geometry& g, const double* x, double* y, cudaStream_t s);
void launch_atb_matched_exact_f64(Geometry& g, const double* y, double* x, cudaStream_t s);
void launch_atb_voxel_f64(Geometry& g, const double* y, double* x, cudaStream_t s);

// f32 performance path (kernels_f32.cu)
void ax_f32(Geometry& g, const float* x, float* y, cudaStream_t s);
void ax_residual_f32(Geometry& g, const float* x, const float* b, double* d_out, cudaStream_t s);
// y1 = A x1 and y2 = A x2 in one pass (f32 Joseph, whole-volume handles): the positions and
// weights are computed once for both volumes; each output is bit-identical to ax_f32's
bool ax2_f32_supported(const Geometry& g);
void ax2_f32(Geometry& g, const float* x1, float* y1, const float* x2, float* y2, cudaStream_t s);
void atb_matched_f32(Geometry& g, const float* y, float* x, cudaStream_t s);
void atb_voxel_f32(Geometry& g, const float* y, float* x, cudaStream_t s);

// operator dispatch (ops.cpp): projector model x precision x variant
template <class T>
void op_ax(Geometry& g, const T* x, T* y, cudaStream_t s);
template <class T>
void op_atb(Geometry& g, int variant, const T* y, T* x, cudaStream_t s);

// Siddon exact-length projector and its transpose (siddon.cu, --fmad=false)
void siddon_ax_zrays_f32(const Geometry& g, const float* x, float* y, cudaStream_t s);
void siddon_atb_zrays_f32(Geometry& g, const float* y, float* x, cudaStream_t s);
template <class T>
void siddon_ax(const Geometry& g, const T* x, T* y, cudaStream_t s);
template <class T>
void siddon_atb(Geometry& g, const T* y, T* x, cudaStream_t s);

// phantom (stencils.cu)
template <class T>
void add_noise(size_t n, const T* in, double i0, double sigma, uint64_t seed, T* out);  // noise.cpp, host
void launch_phantom_f32(int kind, int n, float* out, cudaStream_t s);  // kind: PhantomKind order
void launch_phantom_f64(int kind, int n, double* out, cudaStream_t s);

// ---- BLAS-1 (blas1.cu): deterministic fp64 reductions ----------------------------------
constexpr int kRedBlocks = 592;   // 4 x 148 SMs; fixed => fixed summation order
constexpr int kRedThreads = 256;
constexpr int kRedSlots = 8;      // result slots per workspace

struct RedWork {
    double* partials;  // kRedBlocks * kRedSlots
    double* results;   // kRedSlots
};
RedWork red_work(Geometry* g);             // lazily allocated in g->red
RedWork red_work_global(cudaStream_t s);   // for handle-free BLAS-1 entry points

enum class RedOp { dot, nrm2sq, diff_nrm2sq, axpy_nrm2sq, xpby, lincomb_nrm2sq };
template <class T>
void reduce_dot(size_t n, const T* a, const T* b, double* d_res, RedWork w, cudaStream_t s);
template <class T>
void reduce_diff_nrm2sq(size_t n, const T* a, const T* b, double* d_res, RedWork w, cudaStream_t s);
template <class T>  // y += alpha*x; res = ||y||^2
void axpy_nrm2sq(size_t n, double alpha, const T* x, T* y, double* d_res, RedWork w, cudaStream_t s);
template <class T>
void axpy(size_t n, double alpha, const T* x, T* y, cudaStream_t s);
template <class T>  // y = x + beta*y
void xpby(size_t n, const T* x, double beta, T* y, cudaStream_t s);
template <class T>
void scal(size_t n, double alpha, T* x, cudaStream_t s);
template <class T>  // y = alpha*x
void scale_copy(size_t n, double alpha, const T* x, T* y, cudaStream_t s);
template <class T>  // x += c1*w (old w); w = v - c2*w     (solvers.hpp:114-116)
void lsqr_update(size_t n, double c1, double c2, T* x, T* w, const T* v, cudaStream_t s);
template <class T>  // hbar = h - c1*hbar; x += c2*hbar; h = v - c3*h   (solvers.hpp:201-204)
void lsmr_update(size_t n, double c1, double c2, double c3, T* x, T* h, T* hbar, const T* v, cudaStream_t s);
template <class T>  // r = b - ax, res = ||r||^2
void sub_nrm2sq(size_t n, const T* b, const T* ax, T* r, double* d_res, RedWork w, cudaStream_t s);
template <class T>  // x = 1 / max(x, floor)
void inv_floor(size_t n, double floor, T* x, cudaStream_t s);
template <class T>  // out = a .* b
void mul(size_t n, const T* a, const T* b, T* out, cudaStream_t s);
template <class T>  // x += a .* b
void add_mul(size_t n, const T* a, const T* b, T* x, cudaStream_t s);
template <class T>  // out[i] = max|x|  (fp64)
void reduce_absmax(size_t n, const T* x, double* d_res, RedWork w, cudaStream_t s);
// block Gram-Schmidt pieces (krylov.hpp:21-31, gmres.hpp:33-39): coef[i] = <basis_i, w>
template <class T>
void block_dot(size_t n, int m, const T* basis, size_t ld, const T* w, double* d_coef, double* scratch, cudaStream_t s);
template <class T>  // w += sum_i alpha * coef[i] * basis_i   (coef on device)
void block_axpy(size_t n, int m, double alpha, const double* d_coef, const T* basis, size_t ld, T* w, cudaStream_t s);
template <class T>
void fill(size_t n, T v, T* x, cudaStream_t s);
// fixed-order final reduction of n fp64 partials (one block) -> *d_out
void finish_sum(const double* partials, int n, double* d_out, cudaStream_t s);
void finish_max(const double* partials, int n, double* d_out, cudaStream_t s);

// gradient / TV stencils (stencils.cu)
// z-slab halos: x_above = the next rank's first slice (null: this slab ends the volume);
// gzw_below = the previous rank's last slice of (lam w .* gz); has_above = not the last slab
template <class T>  // out{x,y,z} = scale[i] * (D x)_axis ; scale may be null (=1)
void gradient_scaled(int nx, int ny, int nz, const T* x, const T* scale, double lam, T* gx, T* gy, T* gz, cudaStream_t s,
                     const T* x_above = nullptr);
template <class T>  // out += D^T (lam * w .* g)
void gradient_adjoint_scaled_add(int nx, int ny, int nz, const T* gx, const T* gy, const T* gz, const T* w, double lam,
                                 T* out, cudaStream_t s, const T* gzw_below = nullptr, bool has_above = false);
template <class T>  // w = (|Dx|^2 + eps^2)^(-1/4)
void tv_weights(int nx, int ny, int nz, const T* x, double eps, T* w, cudaStream_t s, const T* x_above = nullptr);

// ---- communicator ----------------------------------------------------------------------
struct Comm {
    ctk_comm_callbacks cb{};
    void* nccl_comm = nullptr;  // when NCCL-backed
    DevBuf gather;              // [nranks][m] staging of comm_sum_vector
};
void comm_allreduce(Comm* c, void* d_buf, size_t count, int dtype, cudaStream_t s);
double comm_sum_scalar(Comm* c, double v);  // rank-ordered sum of per-rank partials
double comm_max_scalar(Comm* c, double v);
std::vector<double> comm_allgather_scalar(Comm* c, double v);  // every rank's value, rank order
// d_v[0..m) <- rank-ordered sum over ranks of every rank's d_v, on stream s: one collective
// for the whole vector (CGS2 coefficients), no host round trip
void comm_sum_vector(Comm* c, double* d_v, int m, cudaStream_t s);
void rank_sum(const double* gathered, int nranks, int m, double* d_out, cudaStream_t s);

// ---- band-sharded range of z-slab sharding (bands.cpp) ----------------------------------
void slab_rows(int mode, int nx, int ny, int nz, int nv, double h, double du, double dso, double dod, int z0, int n,
               int& r0, int& r1);
void slab_rows(const Geometry& g, int z0, int n, int& r0, int& r1);  // rows a z-slab's rays reach
void band_partition(int mode, int nx, int ny, int nz, int nv, double h, double du, double dso, double dod, int nranks,
                    const int* z0s, const int* ns, int* t0, int* t1, int* o0, int* o1);
template <class T>
struct BandSum {
    struct Src {
        const T* p;
        int r0, r1;  // global rows covered
        int rp, roff;  // rows per view in the buffer, global row of its first row
    } src[32];
    int n;
    int o0, o1;  // this rank's owned rows
};
template <class T>
void band_sum(const Geometry& g, const BandSum<T>& bs, T* y, cudaStream_t s);
// A x partials -> owners (rank-ordered sums, other held rows zeroed), in place
template <class T>
void band_reduce(Geometry& g, T* y, cudaStream_t s);
// y with the held rows other ranks own filled in (for A^T b); returns the handle's scratch
template <class T>
const T* band_halo(Geometry& g, const T* y, cudaStream_t s);
void comm_exchange(Comm* c, const std::vector<ctk_p2p_op>& ops, int dtype, cudaStream_t s);

uint64_t launch_count();

}  // namespace ctkb
