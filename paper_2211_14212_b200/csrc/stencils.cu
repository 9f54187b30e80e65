// 7-point stencils of the reweighted-TV operator (HBM-bound, one pass each):
//   gradient           gradient.hpp:9-27      forward differences, zero on the far face
//   gradient_adjoint   gradient.hpp:29-54     exact transpose (fixed term order)
//   tv_weights         tv.hpp:28-43           w = (|Dx|^2 + eps^2)^(-1/4)
// plus the synthetic Shepp-Logan input (phantom.hpp:74-145) used by the bench.
#include "ctk_internal.h"

namespace ctkb {
namespace {

__device__ __forceinline__ void unpack(size_t id, int nx, int ny, int& i, int& j, int& k) {
    i = int(id % nx);
    j = int((id / nx) % ny);
    k = int(id / (size_t(nx) * ny));
}

template <class T>
__global__ void k_gradient_scaled(int nx, int ny, int nz, const T* __restrict__ x, const T* __restrict__ w, T lam,
                                  T* __restrict__ gx, T* __restrict__ gy, T* __restrict__ gz,
                                  const T* __restrict__ x_above) {
    const size_t n = size_t(nx) * ny * nz;
    for (size_t id = size_t(blockIdx.x) * blockDim.x + threadIdx.x; id < n; id += size_t(gridDim.x) * blockDim.x) {
        int i, j, k;
        unpack(id, nx, ny, i, j, k);
        const T v = x[id];
        const T dx = (i + 1 < nx) ? x[id + 1] - v : T(0);
        const T dy = (j + 1 < ny) ? x[id + nx] - v : T(0);
        // z-slab: the top slice differences against the next rank's first slice
        const T dz = (k + 1 < nz) ? x[id + size_t(nx) * ny] - v
                                  : (x_above ? x_above[size_t(i) + size_t(nx) * j] - v : T(0));
        const T s = w ? lam * w[id] : T(1);  // stack_weighted_gradient: s = lam * w_i (operators.hpp:167)
        gx[id] = s * dx;
        gy[id] = s * dy;
        gz[id] = s * dz;
    }
}

template <class T>
__global__ void k_gradient_adjoint_add(int nx, int ny, int nz, const T* __restrict__ gx, const T* __restrict__ gy,
                                       const T* __restrict__ gz, const T* __restrict__ w, T lam, T* __restrict__ out,
                                       const T* __restrict__ gzw_below, int has_above) {
    const size_t n = size_t(nx) * ny * nz;
    const size_t sy = size_t(nx), sz = size_t(nx) * ny;
    for (size_t id = size_t(blockIdx.x) * blockDim.x + threadIdx.x; id < n; id += size_t(gridDim.x) * blockDim.x) {
        int i, j, k;
        unpack(id, nx, ny, i, j, k);
        // the weighted field g' = (lam * w) .* g is formed on the fly (operators.hpp:176-181)
        auto sc = [&](size_t q) { return w ? lam * w[q] : T(1); };
        T acc = 0;
        if (i > 0) acc += sc(id - 1) * gx[id - 1];
        if (i + 1 < nx) acc -= sc(id) * gx[id];
        if (j > 0) acc += sc(id - sy) * gy[id - sy];
        if (j + 1 < ny) acc -= sc(id) * gy[id];
        // z-slab: the previous rank's top-slice term (already weighted) and this rank's top
        // slice, whose difference exists unless this is the last slab
        if (k > 0) acc += sc(id - sz) * gz[id - sz];
        else if (gzw_below) acc += gzw_below[size_t(i) + size_t(nx) * j];
        if (k + 1 < nz || has_above) acc -= sc(id) * gz[id];
        out[id] += acc;
    }
}

template <class T>
__global__ void k_tv_weights(int nx, int ny, int nz, const T* __restrict__ x, double eps, T* __restrict__ w,
                             const T* __restrict__ x_above) {
    const size_t n = size_t(nx) * ny * nz;
    for (size_t id = size_t(blockIdx.x) * blockDim.x + threadIdx.x; id < n; id += size_t(gridDim.x) * blockDim.x) {
        if (eps == 0.0) {
            w[id] = T(1);
            continue;
        }
        int i, j, k;
        unpack(id, nx, ny, i, j, k);
        const T v = x[id];
        const T dx = (i + 1 < nx) ? x[id + 1] - v : T(0);
        const T dy = (j + 1 < ny) ? x[id + nx] - v : T(0);
        const T dz = (k + 1 < nz) ? x[id + size_t(nx) * ny] - v
                                  : (x_above ? x_above[size_t(i) + size_t(nx) * j] - v : T(0));
        const double m2 = double(dx) * dx + double(dy) * dy + double(dz) * dz;
        w[id] = T(pow(m2 + eps * eps, -0.25));
    }
}

// Synthetic ground truth, make_phantom (phantom.hpp:118-145).  Ellipsoid tables
// (phantom.hpp:57-89; columns cx cy cz ax ay az phi intensity), `contains` (:31-39),
// rasterised on cell centres (:93-112): a grid point sums the intensity of every ellipsoid that contains it, in table
// order, in fp64 with the reference's operation order, then converts to T.
__constant__ double c_sl3d[10][8] = {
    {0.0, 0.0, 0.0, 0.69, 0.92, 0.81, 0.0, 2.0},
    {0.0, -0.0184, 0.0, 0.6624, 0.874, 0.78, 0.0, -0.8},
    {0.22, 0.0, 0.0, 0.11, 0.31, 0.22, -18.0, -0.2},
    {-0.22, 0.0, 0.0, 0.16, 0.41, 0.28, 18.0, -0.2},
    {0.0, 0.35, -0.15, 0.21, 0.25, 0.41, 0.0, 0.1},
    {0.0, 0.1, 0.25, 0.046, 0.046, 0.05, 0.0, 0.1},
    {0.0, -0.1, 0.25, 0.046, 0.046, 0.05, 0.0, 0.1},
    {-0.08, -0.605, 0.0, 0.046, 0.023, 0.05, 0.0, 0.1},
    {0.0, -0.605, 0.0, 0.023, 0.023, 0.02, 0.0, 0.1},
    {0.06, -0.605, 0.0, 0.023, 0.046, 0.02, 0.0, 0.1},
};
__constant__ double c_sl2d[10][8] = {
    {0.0, 0.0, 0.0, 0.69, 0.92, 1.0, 0.0, 2.0},
    {0.0, -0.0184, 0.0, 0.6624, 0.874, 1.0, 0.0, -0.98},
    {0.22, 0.0, 0.0, 0.11, 0.31, 1.0, -18.0, -0.02},
    {-0.22, 0.0, 0.0, 0.16, 0.41, 1.0, 18.0, -0.02},
    {0.0, 0.35, 0.0, 0.21, 0.25, 1.0, 0.0, 0.01},
    {0.0, 0.1, 0.0, 0.046, 0.046, 1.0, 0.0, 0.01},
    {0.0, -0.1, 0.0, 0.046, 0.046, 1.0, 0.0, 0.01},
    {-0.08, -0.605, 0.0, 0.046, 0.023, 1.0, 0.0, 0.01},
    {0.0, -0.605, 0.0, 0.023, 0.023, 1.0, 0.0, 0.01},
    {0.06, -0.605, 0.0, 0.023, 0.046, 1.0, 0.0, 0.01},
};

template <class T, bool FLAT>
__global__ void k_ellipsoids(int n, int nz, const double2* __restrict__ rot, T* __restrict__ out) {
    const size_t nn = size_t(n) * n * nz;
    for (size_t id = size_t(blockIdx.x) * blockDim.x + threadIdx.x; id < nn; id += size_t(gridDim.x) * blockDim.x) {
        int i, j, k;
        unpack(id, n, n, i, j, k);
        const double z = nz == 1 ? 0.0 : double(2 * k + 1 - nz) / nz;
        const double y = double(2 * j + 1 - n) / n;
        const double x = double(2 * i + 1 - n) / n;
        double v = 0.0;
        for (int e = 0; e < 10; ++e) {
            const double* p = FLAT ? c_sl2d[e] : c_sl3d[e];
            const double c = rot[e].x, s = rot[e].y;
            const double dx = x - p[0], dy = y - p[1], dz = z - p[2];
            const double xr = __dadd_rn(__dmul_rn(c, dx), __dmul_rn(s, dy));
            const double yr = __dadd_rn(__dmul_rn(-s, dx), __dmul_rn(c, dy));
            const double uu = xr / p[3], vv = yr / p[4], ww = dz / p[5];
            if (__dadd_rn(__dadd_rn(__dmul_rn(uu, uu), __dmul_rn(vv, vv)), __dmul_rn(ww, ww)) <= 1.0) v += p[7];
        }
        out[id] = T(v);
    }
}

// piecewise_blocks (phantom.hpp:133-142): two nested axis-aligned squares, one slice.
template <class T>
__global__ void k_blocks(int n, T* __restrict__ out) {
    const size_t nn = size_t(n) * n;
    const int lo1 = n / 4, hi1 = (3 * n) / 4, lo2 = (3 * n) / 8, hi2 = (5 * n) / 8;
    for (size_t id = size_t(blockIdx.x) * blockDim.x + threadIdx.x; id < nn; id += size_t(gridDim.x) * blockDim.x) {
        const int i = int(id % size_t(n)), j = int(id / size_t(n));
        T v = 0;
        if (i >= lo1 && i < hi1 && j >= lo1 && j < hi1) v += T(0.5);
        if (i >= lo2 && i < hi2 && j >= lo2 && j < hi2) v += T(0.5);
        out[id] = v;
    }
}

template <class T>
void make_phantom(int kind, int n, T* out, cudaStream_t s) {
    const int nz = kind == 0 ? n : 1;
    const size_t nn = size_t(n) * n * nz;
    const size_t blocks = std::min<size_t>((nn + 255) / 256, size_t(148) * 32);
    if (kind == 2) {
        k_blocks<T><<<unsigned(blocks), 256, 0, s>>>(n, out);
        after_launch("k_blocks");
        return;
    }
    // rotation cos/sin from the host libm, like the reference (phantom.hpp:33); both
    // tables share the same angles
    double2 rot[10];
    const double pi = 3.14159265358979323846;
    const double ang[10] = {0.0, 0.0, -18.0, 18.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int e = 0; e < 10; ++e) {
        const double phi = ang[e] * pi / 180.0;
        rot[e] = make_double2(std::cos(phi), std::sin(phi));
    }
    DevBuf d_rot;
    d_rot.ensure(sizeof(rot));
    CTK_CUDA(cudaMemcpyAsync(d_rot.p, rot, sizeof(rot), cudaMemcpyHostToDevice, s));
    if (kind == 0) k_ellipsoids<T, false><<<unsigned(blocks), 256, 0, s>>>(n, nz, d_rot.as<double2>(), out);
    else k_ellipsoids<T, true><<<unsigned(blocks), 256, 0, s>>>(n, nz, d_rot.as<double2>(), out);
    after_launch("k_ellipsoids");
    CTK_CUDA(cudaStreamSynchronize(s));  // d_rot is freed on return
}

size_t grid_for(size_t n) { return std::min<size_t>((n + 255) / 256, size_t(148) * 16); }

}  // namespace

void launch_phantom_f32(int kind, int n, float* out, cudaStream_t s) { make_phantom<float>(kind, n, out, s); }
void launch_phantom_f64(int kind, int n, double* out, cudaStream_t s) { make_phantom<double>(kind, n, out, s); }

template <class T>
void gradient_scaled(int nx, int ny, int nz, const T* x, const T* scale, double lam, T* gx, T* gy, T* gz, cudaStream_t s,
                     const T* x_above) {
    const size_t n = size_t(nx) * ny * nz;
    k_gradient_scaled<T><<<unsigned(grid_for(n)), 256, 0, s>>>(nx, ny, nz, x, scale, T(lam), gx, gy, gz, x_above);
    after_launch("k_gradient_scaled");
}
template <class T>
void gradient_adjoint_scaled_add(int nx, int ny, int nz, const T* gx, const T* gy, const T* gz, const T* w, double lam,
                                 T* out, cudaStream_t s, const T* gzw_below, bool has_above) {
    const size_t n = size_t(nx) * ny * nz;
    k_gradient_adjoint_add<T><<<unsigned(grid_for(n)), 256, 0, s>>>(nx, ny, nz, gx, gy, gz, w, T(lam), out, gzw_below,
                                                                     has_above ? 1 : 0);
    after_launch("k_gradient_adjoint_add");
}
template <class T>
void tv_weights(int nx, int ny, int nz, const T* x, double eps, T* w, cudaStream_t s, const T* x_above) {
    const size_t n = size_t(nx) * ny * nz;
    k_tv_weights<T><<<unsigned(grid_for(n)), 256, 0, s>>>(nx, ny, nz, x, eps, w, x_above);
    after_launch("k_tv_weights");
}

template void gradient_scaled<float>(int, int, int, const float*, const float*, double, float*, float*, float*, cudaStream_t,
                                     const float*);
template void gradient_scaled<double>(int, int, int, const double*, const double*, double, double*, double*, double*,
                                      cudaStream_t, const double*);
template void gradient_adjoint_scaled_add<float>(int, int, int, const float*, const float*, const float*, const float*,
                                                 double, float*, cudaStream_t, const float*, bool);
template void gradient_adjoint_scaled_add<double>(int, int, int, const double*, const double*, const double*,
                                                  const double*, double, double*, cudaStream_t, const double*, bool);
template void tv_weights<float>(int, int, int, const float*, double, float*, cudaStream_t, const float*);
template void tv_weights<double>(int, int, int, const double*, double, double*, cudaStream_t, const double*);

}  // namespace ctkb
