// Fused single-pass BLAS-1 for the solvers (types.hpp:136-158 and the inline vector
// loops of solvers.hpp / krylov.hpp / gmres.hpp).  HBM-bound; every reduction accumulates
// in fp64 over a FIXED partition (kRedBlocks contiguous chunks, fixed shuffle tree,
// fixed-order finish) so results are bitwise run-to-run deterministic
// (test_solvers.cpp:436-451 asks for identical logs).  Vectorised 16-byte loads when the
// pointers allow it.
#include "ctk_internal.h"
#include "reduce.cuh"

namespace ctkb {
namespace {

__global__ void k_finish_sum(const double* __restrict__ p, int n, double* __restrict__ out) {
    double v = 0.0;
    // each thread sums a contiguous run, then the fixed block tree
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int b = threadIdx.x * per, e = min(n, b + per);
    for (int i = b; i < e; ++i) v += p[i];
    v = block_sum(v);
    if (threadIdx.x == 0) *out = v;
}

__global__ void k_finish_max(const double* __restrict__ p, int n, double* __restrict__ out) {
    double v = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) v = fmax(v, p[i]);
    v = block_max(v);
    if (threadIdx.x == 0) *out = v;
}

template <class T>
struct Pair2 {
    T a, b;
};
template <class T>
__device__ __forceinline__ Pair2<T> make_pair2(T a, T b) { return {a, b}; }

struct Chunk {
    size_t b, e;
};
__device__ __forceinline__ Chunk my_chunk(size_t n) {
    const size_t per = (n + gridDim.x - 1) / gridDim.x;
    const size_t b = min(n, size_t(blockIdx.x) * per);
    return {b, min(n, b + per)};
}

// Four independent partial sums per thread over eight elements per iteration (i, i+B, ...,
// i+7B of the block's chunk): eight loads per operand in flight instead of one -- with 4
// resident blocks of 256 threads per SM a single load each keeps only ~8 KB in flight, well
// short of what HBM latency x bandwidth needs.  The combination order is fixed, so results
// stay run-to-run bitwise identical.
template <class T, class F>
__device__ __forceinline__ double chunk_reduce(size_t n, F f) {
    const Chunk c = my_chunk(n);
    const size_t B = blockDim.x;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    size_t i = c.b + threadIdx.x;
    for (; i + 7 * B < c.e; i += 8 * B) {  // eight elements' loads in flight
        const double v0 = f(i), v1 = f(i + B), v2 = f(i + 2 * B), v3 = f(i + 3 * B);
        const double v4 = f(i + 4 * B), v5 = f(i + 5 * B), v6 = f(i + 6 * B), v7 = f(i + 7 * B);
        a0 += v0 + v4;
        a1 += v1 + v5;
        a2 += v2 + v6;
        a3 += v3 + v7;
    }
    for (; i < c.e; i += B) a0 += f(i);
    return block_sum((a0 + a1) + (a2 + a3));
}

// The same with a store per element: ld(i) reads element i's operands, st(i, v) writes it
// and returns its contribution.  All four elements' loads are issued before any store (the
// operations are elementwise, so this reorders nothing that could alias).
template <class T, class LD, class ST>
__device__ __forceinline__ double chunk_reduce_st(size_t n, LD ld, ST st) {
    const Chunk c = my_chunk(n);
    const size_t B = blockDim.x;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    size_t i = c.b + threadIdx.x;
    for (; i + 3 * B < c.e; i += 4 * B) {
        const auto v0 = ld(i), v1 = ld(i + B), v2 = ld(i + 2 * B), v3 = ld(i + 3 * B);
        a0 += st(i, v0);
        a1 += st(i + B, v1);
        a2 += st(i + 2 * B, v2);
        a3 += st(i + 3 * B, v3);
    }
    for (; i < c.e; i += B) a0 += st(i, ld(i));
    return block_sum((a0 + a1) + (a2 + a3));
}

template <class T>
__global__ void k_dot(size_t n, const T* __restrict__ a, const T* __restrict__ b, double* __restrict__ part) {
    const double r = chunk_reduce<T>(n, [&](size_t i) { return double(a[i]) * double(b[i]); });
    if (threadIdx.x == 0) part[blockIdx.x] = r;
}

template <class T>
__global__ void k_diff_nrm2sq(size_t n, const T* __restrict__ a, const T* __restrict__ b, double* __restrict__ part) {
    const double r = chunk_reduce<T>(n, [&](size_t i) {
        const double d = double(a[i]) - double(b[i]);
        return d * d;
    });
    if (threadIdx.x == 0) part[blockIdx.x] = r;
}

template <class T>
__global__ void k_axpy_nrm2sq(size_t n, T alpha, const T* __restrict__ x, T* __restrict__ y, double* __restrict__ part) {
    const double r = chunk_reduce_st<T>(
        n, [&](size_t i) { return make_pair2(x[i], y[i]); },
        [&](size_t i, Pair2<T> p) {
            const T v = p.b + alpha * p.a;
            y[i] = v;
            return double(v) * double(v);
        });
    if (threadIdx.x == 0) part[blockIdx.x] = r;
}

// r = b - ax; partial of ||r||^2 (SIRT residual, solvers.hpp:280-282)
template <class T>
__global__ void k_sub_nrm2sq(size_t n, const T* __restrict__ b, const T* __restrict__ ax, T* __restrict__ r,
                             double* __restrict__ part) {
    const double v = chunk_reduce_st<T>(
        n, [&](size_t i) { return make_pair2(b[i], ax[i]); },
        [&](size_t i, Pair2<T> p) {
            const T d = p.a - p.b;
            r[i] = d;
            return double(d) * double(d);
        });
    if (threadIdx.x == 0) part[blockIdx.x] = v;
}

template <class T>
__global__ void k_absmax(size_t n, const T* __restrict__ x, double* __restrict__ part) {
    const Chunk c = my_chunk(n);
    double m = 0.0;
    for (size_t i = c.b + threadIdx.x; i < c.e; i += blockDim.x) m = fmax(m, fabs(double(x[i])));
    m = block_max(m);
    if (threadIdx.x == 0) part[blockIdx.x] = m;
}

// Elementwise maps: F::load(i) reads element i's operands, F::store(i, v) writes its
// results.  Four grid-stride elements per iteration with all loads issued before the stores
// (four loads per operand in flight; elementwise, so nothing that can alias is reordered).
template <class T, class F>
__global__ void k_map(size_t n, F f) {
    const size_t S = size_t(gridDim.x) * blockDim.x;
    size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + 3 * S < n; i += 4 * S) {
        const auto v0 = f.load(i), v1 = f.load(i + S), v2 = f.load(i + 2 * S), v3 = f.load(i + 3 * S);
        f.store(i, v0);
        f.store(i + S, v1);
        f.store(i + 2 * S, v2);
        f.store(i + 3 * S, v3);
    }
    for (; i < n; i += S) f.store(i, f.load(i));
}

template <class T>
struct V1 {
    T a;
};
template <class T>
struct V2 {
    T a, b;
};
template <class T>
struct V3 {
    T a, b, c;
};
template <class T>
struct V4 {
    T a, b, c, d;
};

template <class T>
struct AxpyF {  // y += a x
    T a;
    const T* x;
    T* y;
    __device__ V2<T> load(size_t i) const { return {x[i], y[i]}; }
    __device__ void store(size_t i, V2<T> v) const { y[i] = v.b + a * v.a; }
};
template <class T>
struct XpbyF {  // y = x + b y
    const T* x;
    T b;
    T* y;
    __device__ V2<T> load(size_t i) const { return {x[i], y[i]}; }
    __device__ void store(size_t i, V2<T> v) const { y[i] = v.a + b * v.b; }
};
template <class T>
struct ScalF {
    T a;
    T* x;
    __device__ V1<T> load(size_t i) const { return {x[i]}; }
    __device__ void store(size_t i, V1<T> v) const { x[i] = v.a * a; }
};
template <class T>
struct ScaleCopyF {
    T a;
    const T* x;
    T* y;
    __device__ V1<T> load(size_t i) const { return {x[i]}; }
    __device__ void store(size_t i, V1<T> v) const { y[i] = a * v.a; }
};
template <class T>
struct LsqrF {
    T c1, c2;
    T* x;
    T* w;
    const T* v;
    __device__ V3<T> load(size_t i) const { return {x[i], w[i], v[i]}; }
    __device__ void store(size_t i, V3<T> e) const {
        x[i] = e.a + c1 * e.b;
        w[i] = e.c - c2 * e.b;
    }
};
template <class T>
struct LsmrF {
    T c1, c2, c3;
    T* x;
    T* h;
    T* hbar;
    const T* v;
    __device__ V4<T> load(size_t i) const { return {h[i], hbar[i], x[i], v[i]}; }
    __device__ void store(size_t i, V4<T> e) const {
        const T hb = e.a - c1 * e.b;
        hbar[i] = hb;
        x[i] = e.c + c2 * hb;
        h[i] = e.d - c3 * e.a;
    }
};
template <class T>
struct InvFloorF {  // x = 1 / max(x, floor)   (solvers.hpp:257-263)
    T floor;
    T* x;
    __device__ V1<T> load(size_t i) const { return {x[i]}; }
    __device__ void store(size_t i, V1<T> v) const { x[i] = T(1) / (v.a > floor ? v.a : floor); }
};
template <class T>
struct MulF {  // out = a .* b
    const T* a;
    const T* b;
    T* out;
    __device__ V2<T> load(size_t i) const { return {a[i], b[i]}; }
    __device__ void store(size_t i, V2<T> v) const { out[i] = v.a * v.b; }
};
template <class T>
struct AddMulF {  // x += a .* b
    const T* a;
    const T* b;
    T* x;
    __device__ V3<T> load(size_t i) const { return {a[i], b[i], x[i]}; }
    __device__ void store(size_t i, V3<T> v) const { x[i] = v.c + v.a * v.b; }
};
template <class T>
struct FillF {
    T v;
    T* x;
    __device__ V1<T> load(size_t) const { return {v}; }
    __device__ void store(size_t i, V1<T> e) const { x[i] = e.a; }
};

template <class T, class F>
void run_map(size_t n, F f, cudaStream_t s, const char* what) {
    if (n == 0) return;
    const size_t blocks = std::min<size_t>((n + 255) / 256, size_t(148) * 16);
    k_map<T, F><<<unsigned(blocks), 256, 0, s>>>(n, f);
    after_launch(what);
}

// block_dot: coef[q] = <basis_q, w>, partials[q][blk] then a fixed-order finish per q.
// Basis vectors in groups of BD_G: w is read once per group (not once per vector) and each
// thread has 1 + BD_G independent loads in flight per element.
constexpr int BD_G = 8;
// One group of G basis vectors over the block's chunk: two elements per iteration, all
// 2 * (1 + G) loads issued before the FMAs.
template <int G, class T>
__device__ __forceinline__ void block_dot_group(const Chunk& c, const T* __restrict__ bq, size_t ld,
                                                const T* __restrict__ w, double* acc) {
    const size_t B = blockDim.x;
    size_t i = c.b + threadIdx.x;
    for (; i + B < c.e; i += 2 * B) {
        const double w0 = double(__ldg(w + i)), w1 = double(__ldg(w + i + B));
        T b0[G], b1[G];
#pragma unroll
        for (int j = 0; j < G; ++j) {
            b0[j] = __ldg(bq + size_t(j) * ld + i);
            b1[j] = __ldg(bq + size_t(j) * ld + i + B);
        }
#pragma unroll
        for (int j = 0; j < G; ++j) acc[j] += double(b0[j]) * w0 + double(b1[j]) * w1;
    }
    if (i < c.e) {
        const double w0 = double(__ldg(w + i));
#pragma unroll
        for (int j = 0; j < G; ++j) acc[j] += double(__ldg(bq + size_t(j) * ld + i)) * w0;
    }
}

template <class T>
__global__ void k_block_dot(size_t n, int m, const T* __restrict__ basis, size_t ld, const T* __restrict__ w,
                            double* __restrict__ part) {
    const Chunk c = my_chunk(n);
    for (int q0 = 0; q0 < m; q0 += BD_G) {
        const int g = min(BD_G, m - q0);
        const T* bq = basis + size_t(q0) * ld;
        double acc[BD_G];
#pragma unroll
        for (int j = 0; j < BD_G; ++j) acc[j] = 0.0;
        switch (g) {  // a group of exactly g vectors: no idle or duplicated loads
            case 1: block_dot_group<1>(c, bq, ld, w, acc); break;
            case 2: block_dot_group<2>(c, bq, ld, w, acc); break;
            case 3: block_dot_group<3>(c, bq, ld, w, acc); break;
            case 4: block_dot_group<4>(c, bq, ld, w, acc); break;
            case 5: block_dot_group<5>(c, bq, ld, w, acc); break;
            case 6: block_dot_group<6>(c, bq, ld, w, acc); break;
            case 7: block_dot_group<7>(c, bq, ld, w, acc); break;
            default: block_dot_group<BD_G>(c, bq, ld, w, acc); break;
        }
#pragma unroll
        for (int j = 0; j < BD_G; ++j) {
            if (j < g) {  // uniform across the block
                const double v = block_sum(acc[j]);
                if (threadIdx.x == 0) part[size_t(q0 + j) * gridDim.x + blockIdx.x] = v;
            }
        }
    }
}

__global__ void k_finish_many(const double* __restrict__ part, int nblk, double* __restrict__ out) {
    const double* p = part + size_t(blockIdx.x) * nblk;
    double v = 0.0;
    const int per = (nblk + blockDim.x - 1) / blockDim.x;
    const int b = threadIdx.x * per, e = min(nblk, b + per);
    for (int i = b; i < e; ++i) v += p[i];
    v = block_sum(v);
    if (threadIdx.x == 0) out[blockIdx.x] = v;
}

// w += alpha * sum_q coef[q] basis_q, accumulated in T in q order (as the sequence of
// per-vector axpys it replaces); the scaled coefficients are staged in shared memory and the
// basis loads of a group of BD_G vectors are issued together.
constexpr int BA_MAXM = 1024;
template <class T>
__global__ void k_block_axpy(size_t n, int m, double alpha, const double* __restrict__ coef, const T* __restrict__ basis,
                             size_t ld, T* __restrict__ w) {
    __shared__ T cs[BA_MAXM];
    for (int q = threadIdx.x; q < m; q += blockDim.x) cs[q] = T(alpha * coef[q]);
    __syncthreads();
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        T acc = w[i];
        int q0 = 0;
        for (; q0 + BD_G <= m; q0 += BD_G) {  // full groups: all loads issue before the FMAs
            T bv[BD_G];
#pragma unroll
            for (int j = 0; j < BD_G; ++j) bv[j] = __ldg(basis + size_t(q0 + j) * ld + i);
#pragma unroll
            for (int j = 0; j < BD_G; ++j) acc += cs[q0 + j] * bv[j];
        }
        for (; q0 < m; ++q0) acc += cs[q0] * basis[size_t(q0) * ld + i];
        w[i] = acc;
    }
}

}  // namespace

// out[j] = sum_r g[r*m + j] with r ascending: the rank-ordered sum of an all-gathered
// coefficient vector (every rank evaluates the same sequence -> bitwise equal results)
__global__ void k_rank_sum(const double* __restrict__ g, int nranks, int m, double* __restrict__ out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    double acc = 0.0;
    for (int r = 0; r < nranks; ++r) acc += g[size_t(r) * m + j];
    out[j] = acc;
}

void rank_sum(const double* gathered, int nranks, int m, double* d_out, cudaStream_t s) {
    if (m <= 0) return;
    k_rank_sum<<<(m + 127) / 128, 128, 0, s>>>(gathered, nranks, m, d_out);
    after_launch("k_rank_sum");
}

void finish_sum(const double* partials, int n, double* d_out, cudaStream_t s) {
    k_finish_sum<<<1, 256, 0, s>>>(partials, n, d_out);
    after_launch("k_finish_sum");
}
void finish_max(const double* partials, int n, double* d_out, cudaStream_t s) {
    k_finish_max<<<1, 256, 0, s>>>(partials, n, d_out);
    after_launch("k_finish_max");
}

template <class T>
void reduce_dot(size_t n, const T* a, const T* b, double* d_res, RedWork w, cudaStream_t s) {
    k_dot<T><<<kRedBlocks, kRedThreads, 0, s>>>(n, a, b, w.partials);
    after_launch("k_dot");
    finish_sum(w.partials, kRedBlocks, d_res, s);
}
template <class T>
void reduce_diff_nrm2sq(size_t n, const T* a, const T* b, double* d_res, RedWork w, cudaStream_t s) {
    k_diff_nrm2sq<T><<<kRedBlocks, kRedThreads, 0, s>>>(n, a, b, w.partials);
    after_launch("k_diff_nrm2sq");
    finish_sum(w.partials, kRedBlocks, d_res, s);
}
template <class T>
void axpy_nrm2sq(size_t n, double alpha, const T* x, T* y, double* d_res, RedWork w, cudaStream_t s) {
    k_axpy_nrm2sq<T><<<kRedBlocks, kRedThreads, 0, s>>>(n, T(alpha), x, y, w.partials);
    after_launch("k_axpy_nrm2sq");
    finish_sum(w.partials, kRedBlocks, d_res, s);
}
template <class T>
void sub_nrm2sq(size_t n, const T* b, const T* ax, T* r, double* d_res, RedWork w, cudaStream_t s) {
    k_sub_nrm2sq<T><<<kRedBlocks, kRedThreads, 0, s>>>(n, b, ax, r, w.partials);
    after_launch("k_sub_nrm2sq");
    finish_sum(w.partials, kRedBlocks, d_res, s);
}
template <class T>
void inv_floor(size_t n, double floor, T* x, cudaStream_t s) {
    run_map<T>(n, InvFloorF<T>{T(floor), x}, s, "k_inv_floor");
}
template <class T>
void mul(size_t n, const T* a, const T* b, T* out, cudaStream_t s) {
    run_map<T>(n, MulF<T>{a, b, out}, s, "k_mul");
}
template <class T>
void add_mul(size_t n, const T* a, const T* b, T* x, cudaStream_t s) {
    run_map<T>(n, AddMulF<T>{a, b, x}, s, "k_add_mul");
}
template <class T>
void reduce_absmax(size_t n, const T* x, double* d_res, RedWork w, cudaStream_t s) {
    k_absmax<T><<<kRedBlocks, kRedThreads, 0, s>>>(n, x, w.partials);
    after_launch("k_absmax");
    finish_max(w.partials, kRedBlocks, d_res, s);
}
template <class T>
void axpy(size_t n, double alpha, const T* x, T* y, cudaStream_t s) {
    run_map<T>(n, AxpyF<T>{T(alpha), x, y}, s, "k_axpy");
}
template <class T>
void xpby(size_t n, const T* x, double beta, T* y, cudaStream_t s) {
    run_map<T>(n, XpbyF<T>{x, T(beta), y}, s, "k_xpby");
}
template <class T>
void scal(size_t n, double alpha, T* x, cudaStream_t s) {
    run_map<T>(n, ScalF<T>{T(alpha), x}, s, "k_scal");
}
template <class T>
void scale_copy(size_t n, double alpha, const T* x, T* y, cudaStream_t s) {
    run_map<T>(n, ScaleCopyF<T>{T(alpha), x, y}, s, "k_scale_copy");
}
template <class T>
void lsqr_update(size_t n, double c1, double c2, T* x, T* w, const T* v, cudaStream_t s) {
    run_map<T>(n, LsqrF<T>{T(c1), T(c2), x, w, v}, s, "k_lsqr_update");
}
template <class T>
void lsmr_update(size_t n, double c1, double c2, double c3, T* x, T* h, T* hbar, const T* v, cudaStream_t s) {
    run_map<T>(n, LsmrF<T>{T(c1), T(c2), T(c3), x, h, hbar, v}, s, "k_lsmr_update");
}
template <class T>
void fill(size_t n, T v, T* x, cudaStream_t s) {
    run_map<T>(n, FillF<T>{v, x}, s, "k_fill");
}
template <class T>
void block_dot(size_t n, int m, const T* basis, size_t ld, const T* w, double* d_coef, double* scratch, cudaStream_t s) {
    if (m <= 0) return;
    k_block_dot<T><<<kRedBlocks, kRedThreads, 0, s>>>(n, m, basis, ld, w, scratch);
    after_launch("k_block_dot");
    k_finish_many<<<m, 256, 0, s>>>(scratch, kRedBlocks, d_coef);
    after_launch("k_finish_many");
}
template <class T>
void block_axpy(size_t n, int m, double alpha, const double* d_coef, const T* basis, size_t ld, T* w, cudaStream_t s) {
    if (m <= 0) return;
    const size_t blocks = std::min<size_t>((n + 255) / 256, size_t(148) * 16);
    // more than BA_MAXM vectors: consecutive launches over consecutive vector ranges keep
    // the per-element q order
    for (int q0 = 0; q0 < m; q0 += BA_MAXM) {
        k_block_axpy<T><<<unsigned(blocks), 256, 0, s>>>(n, std::min(BA_MAXM, m - q0), alpha, d_coef + q0,
                                                         basis + size_t(q0) * ld, ld, w);
        after_launch("k_block_axpy");
    }
}

// band-sharded range (bands.cpp): y's owned rows <- rank-ordered sum of the partials of
// every source that covers the row; y's other held rows <- 0.  In place: a thread reads the
// local partial of its element before writing it.
template <class T>
__global__ void k_band_sum(BandSum<T> bs, int na, int nu, int w0, int nw, T* __restrict__ y) {
    const size_t n = size_t(na) * nw * nu;
    for (size_t id = size_t(blockIdx.x) * blockDim.x + threadIdx.x; id < n; id += size_t(gridDim.x) * blockDim.x) {
        const int iu = int(id % nu);
        const size_t ar = id / nu;
        const int row = w0 + int(ar % nw), a = int(ar / nw);
        T acc = T(0);
        if (row >= bs.o0 && row < bs.o1) {
            for (int i = 0; i < bs.n; ++i) {
                const auto& sr = bs.src[i];
                if (row >= sr.r0 && row < sr.r1) acc += sr.p[(size_t(a) * sr.rp + size_t(row - sr.roff)) * nu + iu];
            }
        }
        y[id] = acc;
    }
}

template <class T>
void band_sum(const Geometry& g, const BandSum<T>& bs, T* y, cudaStream_t s) {
    const size_t n = g.range();
    const unsigned blocks = unsigned(std::min<size_t>((n + 255) / 256, 148 * 16));
    k_band_sum<T><<<blocks, 256, 0, s>>>(bs, g.na, g.nu, g.w0, g.nw, y);
    after_launch("k_band_sum");
}

#define CTK_INST(T)                                                                                        \
    template void reduce_dot<T>(size_t, const T*, const T*, double*, RedWork, cudaStream_t);              \
    template void reduce_diff_nrm2sq<T>(size_t, const T*, const T*, double*, RedWork, cudaStream_t);      \
    template void axpy_nrm2sq<T>(size_t, double, const T*, T*, double*, RedWork, cudaStream_t);           \
    template void reduce_absmax<T>(size_t, const T*, double*, RedWork, cudaStream_t);                     \
    template void sub_nrm2sq<T>(size_t, const T*, const T*, T*, double*, RedWork, cudaStream_t);          \
    template void inv_floor<T>(size_t, double, T*, cudaStream_t);                                         \
    template void mul<T>(size_t, const T*, const T*, T*, cudaStream_t);                                   \
    template void add_mul<T>(size_t, const T*, const T*, T*, cudaStream_t);                               \
    template void axpy<T>(size_t, double, const T*, T*, cudaStream_t);                                    \
    template void xpby<T>(size_t, const T*, double, T*, cudaStream_t);                                    \
    template void scal<T>(size_t, double, T*, cudaStream_t);                                              \
    template void scale_copy<T>(size_t, double, const T*, T*, cudaStream_t);                              \
    template void lsqr_update<T>(size_t, double, double, T*, T*, const T*, cudaStream_t);                 \
    template void lsmr_update<T>(size_t, double, double, double, T*, T*, T*, const T*, cudaStream_t);     \
    template void fill<T>(size_t, T, T*, cudaStream_t);                                                   \
    template void block_dot<T>(size_t, int, const T*, size_t, const T*, double*, double*, cudaStream_t);  \
    template void block_axpy<T>(size_t, int, double, const double*, const T*, size_t, T*, cudaStream_t); \
    template void band_sum<T>(const Geometry&, const BandSum<T>&, T*, cudaStream_t);
CTK_INST(float)
CTK_INST(double)
#undef CTK_INST

}  // namespace ctkb
