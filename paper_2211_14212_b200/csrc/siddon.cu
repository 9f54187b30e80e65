// Siddon exact-length projector (BASELINE north_star subsystem 1; absent from the
// reference) and its exact transpose, T in {float, double}.
//
// Ray geometry = make_ray (projector.hpp:29-46).  Voxel (i,j,k) is the box
// [(i - n/2) h, (i + 1 - n/2) h] x ...; the weight of (ray, voxel) is the length of the
// ray inside that box (the slab chord of tests/oracles.hpp:89-107 per voxel).  Every plane
// crossing is alpha_a(q) = ((q - n_a/2) h - o_a) * (1/d_a), evaluated identically by the
// forward DDA and by the transpose (min(exit) - max(entry) of the voxel's six crossings),
// so both see bit-identical segment lengths; a ray parallel to an axis belongs to the
// half-open slab containing o_a.  Compiled with --fmad=false: bit-identical to the oracle
// restatement (oracle/ctk_oracle.c) for T=double and T=float.
//   Ax:    thread per ray, 3-D DDA over the crossed voxels, traversal-order accumulation.
//   A^T b: deterministic gather, thread per voxel; candidates = detector footprint of the
//          voxel box; contributions in the (view, row, column) order of the reference's
//          scatter (projector.hpp:187-197).
#include <cfloat>

#include "ctk_internal.h"

namespace ctkb {
namespace {

struct SRay {
    double o[3], d[3], inv[3];
};

__device__ __forceinline__ void s_make_ray(const KGeom& g, double ct, double st, int iu, int iv, SRay& r) {
    const double u = (iu - 0.5 * (g.nu - 1)) * g.du;
    const double v = (iv - 0.5 * (g.nv - 1)) * g.du;
    const double cx = -g.dod * ct, cy = -g.dod * st, cz = 0.0;
    const double px = cx - u * st, py = cy + u * ct, pz = cz + v;
    if (g.mode == CTK_CONE3D) {
        const double sx = g.dso * ct, sy = g.dso * st, sz = 0.0;
        const double dx = px - sx, dy = py - sy, dz = pz - sz;
        const double n = sqrt(dx * dx + dy * dy + dz * dz);
        r.o[0] = sx; r.o[1] = sy; r.o[2] = sz;
        r.d[0] = dx / n; r.d[1] = dy / n; r.d[2] = dz / n;
    } else {
        r.o[0] = px; r.o[1] = py; r.o[2] = pz;
        r.d[0] = -ct; r.d[1] = -st; r.d[2] = 0.0;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) r.inv[a] = r.d[a] != 0.0 ? 1.0 / r.d[a] : 0.0;
}

__device__ __forceinline__ double s_alpha(const SRay& r, int a, int q, int n, double h) {
    return ((q - 0.5 * n) * h - r.o[a]) * r.inv[a];
}

__device__ __forceinline__ int s_slab(double c, int n, double h) { return int(floor(c / h + 0.5 * n)); }

template <class T>
__global__ void k_siddon_ax(KGeom g, const T* __restrict__ vol, T* __restrict__ proj) {
    const int iu = blockIdx.x * blockDim.x + threadIdx.x;
    const int iv = blockIdx.y * blockDim.y + threadIdx.y;
    const int a = blockIdx.z;
    if (iu >= g.nu || iv >= g.nv) return;
    const double2 cs = g.ctst[a];
    SRay r;
    s_make_ray(g, cs.x, cs.y, iu, iv, r);
    const int n3[3] = {g.nx, g.ny, g.nz};
    const double h = g.h;
    double amin = -DBL_MAX, amax = DBL_MAX;
    bool ok = true;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        if (r.d[ax] == 0.0) {
            const int sl = s_slab(r.o[ax], n3[ax], h);
            if (sl < 0 || sl >= n3[ax]) ok = false;
            continue;
        }
        const double e0 = s_alpha(r, ax, 0, n3[ax], h), e1 = s_alpha(r, ax, n3[ax], n3[ax], h);
        amin = fmax(amin, fmin(e0, e1));
        amax = fmin(amax, fmax(e0, e1));
    }
    T acc = 0;
    if (ok && amin < amax) {
        int ix[3], st[3];
        double an[3];
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            if (r.d[ax] == 0.0) {
                ix[ax] = s_slab(r.o[ax], n3[ax], h);
                st[ax] = 0;
                an[ax] = DBL_MAX;
                continue;
            }
            st[ax] = r.d[ax] > 0.0 ? 1 : -1;
            // slab entered at amin (the unique q with entry crossing <= amin < exit crossing)
            int q = min(max(s_slab(r.o[ax] + amin * r.d[ax], n3[ax], h), 0), n3[ax] - 1);
            if (st[ax] > 0) {
                while (q < n3[ax] - 1 && s_alpha(r, ax, q + 1, n3[ax], h) <= amin) ++q;
                while (q > 0 && s_alpha(r, ax, q, n3[ax], h) > amin) --q;
            } else {
                while (q > 0 && s_alpha(r, ax, q, n3[ax], h) <= amin) --q;
                while (q < n3[ax] - 1 && s_alpha(r, ax, q + 1, n3[ax], h) > amin) ++q;
            }
            ix[ax] = q;
            an[ax] = s_alpha(r, ax, st[ax] > 0 ? q + 1 : q, n3[ax], h);
        }
        double acur = amin;
        while (acur < amax) {
            const double anext = fmin(amax, fmin(an[0], fmin(an[1], an[2])));
            const double len = anext - acur;
            if (len > 0.0)
                acc += T(len) * __ldg(vol + size_t(ix[0]) + size_t(n3[0]) * (size_t(ix[1]) + size_t(n3[1]) * ix[2]));
            if (anext >= amax) break;
            bool out = false;
#pragma unroll
            for (int ax = 0; ax < 3; ++ax)
                if (an[ax] == anext) {
                    ix[ax] += st[ax];
                    if (ix[ax] < 0 || ix[ax] >= n3[ax]) out = true;
                    an[ax] = s_alpha(r, ax, st[ax] > 0 ? ix[ax] + 1 : ix[ax], n3[ax], h);
                }
            if (out) break;
            acur = anext;
        }
    }
    proj[size_t(a) * g.nu * g.nv + size_t(iu) + size_t(g.nu) * iv] = acc;
}

// projection of a point onto continuous detector coordinates; false if not in front of
// the cone source (then every pixel is a candidate)
__device__ __forceinline__ bool s_project(const KGeom& g, double ct, double st, double x, double y, double z,
                                          double& fu, double& fv) {
    double u, v;
    if (g.mode == CTK_CONE3D) {
        const double sx = g.dso * ct, sy = g.dso * st;
        const double rx = x - sx, ry = y - sy;
        const double depth = -(rx * ct + ry * st);
        if (!(depth > 1e-9 * g.dso)) return false;
        const double t = (g.dso + g.dod) / depth;
        u = -(sx + t * rx) * st + (sy + t * ry) * ct;
        v = t * z;
    } else {
        u = -x * st + y * ct;
        v = z;
    }
    fu = u / g.du + 0.5 * (g.nu - 1);
    fv = v / g.du + 0.5 * (g.nv - 1);
    return true;
}

template <class T>
__global__ void k_siddon_atb(KGeom g, const T* __restrict__ proj, T* __restrict__ vol) {
    const size_t nvox = size_t(g.nx) * g.ny * g.nz;
    const size_t id = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (id >= nvox) return;
    const int idx3[3] = {int(id % g.nx), int((id / g.nx) % g.ny), int(id / (size_t(g.nx) * g.ny))};
    const int n3[3] = {g.nx, g.ny, g.nz};
    const double h = g.h;
    const double lo3[3] = {(idx3[0] - 0.5 * g.nx) * h, (idx3[1] - 0.5 * g.ny) * h, (idx3[2] - 0.5 * g.nz) * h};
    const size_t frame = size_t(g.nu) * g.nv;
    T acc = 0;
    for (int a = 0; a < g.na; ++a) {
        const double2 cs = g.ctst[a];
        double umin = DBL_MAX, umax = -DBL_MAX, vmin = DBL_MAX, vmax = -DBL_MAX;
        bool all = false;
        for (int q = 0; q < 8; ++q) {
            double fu, fv;
            if (!s_project(g, cs.x, cs.y, lo3[0] + ((q & 1) ? h : 0.0), lo3[1] + ((q & 2) ? h : 0.0),
                           lo3[2] + ((q & 4) ? h : 0.0), fu, fv)) {
                all = true;
                break;
            }
            umin = fmin(umin, fu); umax = fmax(umax, fu);
            vmin = fmin(vmin, fv); vmax = fmax(vmax, fv);
        }
        int iu0 = 0, iu1 = g.nu - 1, iv0 = 0, iv1 = g.nv - 1;
        if (!all) {
            iu0 = max(iu0, int(floor(fmax(umin, -1e9))) - 1);
            iu1 = min(iu1, int(ceil(fmin(umax, 1e9))) + 1);
            if (g.nv > 1) {
                iv0 = max(iv0, int(floor(fmax(vmin, -1e9))) - 1);
                iv1 = min(iv1, int(ceil(fmin(vmax, 1e9))) + 1);
            }
        }
        const T* fr = proj + size_t(a) * frame;
        for (int iv = iv0; iv <= iv1; ++iv)
            for (int iu = iu0; iu <= iu1; ++iu) {
                const T value = __ldg(fr + size_t(iu) + size_t(g.nu) * iv);
                if (value == T(0)) continue;
                SRay r;
                s_make_ray(g, cs.x, cs.y, iu, iv, r);
                double lo = -DBL_MAX, hi = DBL_MAX;
                bool miss = false;
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) {
                    if (r.d[ax] == 0.0) {
                        if (s_slab(r.o[ax], n3[ax], h) != idx3[ax]) miss = true;
                        continue;
                    }
                    const double a0 = s_alpha(r, ax, idx3[ax], n3[ax], h);
                    const double a1 = s_alpha(r, ax, idx3[ax] + 1, n3[ax], h);
                    lo = fmax(lo, fmin(a0, a1));
                    hi = fmin(hi, fmax(a0, a1));
                }
                if (miss || !(hi > lo)) continue;
                acc += T(hi - lo) * value;
            }
    }
    vol[id] = acc;
}

}  // namespace

template <class T>
void siddon_ax(const Geometry& g, const T* x, T* y, cudaStream_t s) {
    dim3 blk(32, 4), grd((g.nu + 31) / 32, (g.nv + 3) / 4, g.na);
    k_siddon_ax<T><<<grd, blk, 0, s>>>(g.kgeom(), x, y);
    after_launch("k_siddon_ax");
}

template <class T>
void siddon_atb(const Geometry& g, const T* y, T* x, cudaStream_t s) {
    const size_t n = g.domain();
    k_siddon_atb<T><<<unsigned((n + 127) / 128), 128, 0, s>>>(g.kgeom(), y, x);
    after_launch("k_siddon_atb");
}

template void siddon_ax<float>(const Geometry&, const float*, float*, cudaStream_t);
template void siddon_ax<double>(const Geometry&, const double*, double*, cudaStream_t);
template void siddon_atb<float>(const Geometry&, const float*, float*, cudaStream_t);
template void siddon_atb<double>(const Geometry&, const double*, double*, cudaStream_t);

}  // namespace ctkb
