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

// zonly: only the rays the f32 slab model leaves out (z-dominant cone rows: |v| > |d_A| of
// the unnormalised ray, f32_common.cuh is_zray); the others are not written
template <class T>
__global__ void k_siddon_ax(KGeom g, const T* __restrict__ vol, T* __restrict__ proj, int zonly) {
    const int iu = blockIdx.x * blockDim.x + threadIdx.x;
    const int iv = blockIdx.y * blockDim.y + threadIdx.y;
    const int a = blockIdx.z;
    if (iu >= g.nu || iv >= g.nv) return;
    if (zonly && !(g.mode == CTK_CONE3D && fabs((iv - 0.5 * (g.nv - 1)) * g.du) > g.colstep[a * g.nu + iu].y)) return;
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

// 1/d of every ray (make_ray, then the reciprocal exactly as s_make_ray forms it), so the
// transpose's candidates cost a 24-byte load instead of a sqrt and six divisions
__global__ void k_siddon_rayinv(KGeom g, double* __restrict__ inv) {
    const int iu = blockIdx.x * blockDim.x + threadIdx.x;
    const int iv = blockIdx.y * blockDim.y + threadIdx.y;
    const int a = blockIdx.z;
    if (iu >= g.nu || iv >= g.nv) return;
    const double2 cs = g.ctst[a];
    SRay r;
    s_make_ray(g, cs.x, cs.y, iu, iv, r);
    double* o = inv + 3 * ((size_t(a) * g.nu + iu) * g.nv + iv);  // [a][iu][iv]
    o[0] = r.inv[0];
    o[1] = r.inv[1];
    o[2] = r.inv[2];
}

// Detector window of the box [lo3, lo3 + h]^3 for one view: the pixel centres inside the
// bounding box of the 8 corner projections (a ray meets the box iff its detector point lies
// in the box's projection).  Only a superset of the hit pixels is needed -- every candidate
// is decided by the exact fp64 slab test -- so the window is computed in f32 with a
// 1e-2-pixel slack (f32 error at |u| <= 2^12 pixels is < 1e-3).  For a cone the four (x, y)
// corners share one depth each: u = w D / depth, v = z D / depth.  false: the box is not
// strictly in front of the source (every pixel is a candidate).
__device__ __forceinline__ bool s_window(const KGeom& g, double ct, double st, const double lo3[3], double h,
                                         int& iu0, int& iu1, int& iv0, int& iv1) {
    float umin = FLT_MAX, umax = -FLT_MAX, vmin = FLT_MAX, vmax = -FLT_MAX;
    const float ctf = float(ct), stf = float(st), hf = float(h);
    const float z0 = float(lo3[2]), z1 = float(lo3[2] + h);
    const float dso = float(g.dso), D = float(g.dso + g.dod);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float x = float(lo3[0]) + ((q & 1) ? hf : 0.f), y = float(lo3[1]) + ((q & 2) ? hf : 0.f);
        const float w = -x * stf + y * ctf;
        if (g.mode == CTK_CONE3D) {
            const float depth = dso - (x * ctf + y * stf);
            if (!(depth > 1e-6f * dso)) return false;
            const float t = D * __frcp_rn(depth);
            umin = fminf(umin, w * t);
            umax = fmaxf(umax, w * t);
            vmin = fminf(vmin, fminf(z0 * t, z1 * t));
            vmax = fmaxf(vmax, fmaxf(z0 * t, z1 * t));
        } else {
            umin = fminf(umin, w);
            umax = fmaxf(umax, w);
            vmin = z0;
            vmax = z1;
        }
    }
    const float idu = float(1.0 / g.du), cu = 0.5f * float(g.nu - 1), cv = 0.5f * float(g.nv - 1), eps = 1e-2f;
    iu0 = max(0, int(ceilf(fmaxf(fmaf(umin, idu, cu - eps), -1e9f))));
    iu1 = min(g.nu - 1, int(floorf(fminf(fmaf(umax, idu, cu + eps), 1e9f))));
    iv0 = 0;
    iv1 = g.nv - 1;
    if (g.nv > 1) {
        iv0 = max(0, int(ceilf(fmaxf(fmaf(vmin, idu, cv - eps), -1e9f))));
        iv1 = min(g.nv - 1, int(floorf(fminf(fmaf(vmax, idu, cv + eps), 1e9f))));
    }
    return true;
}

// Transpose as a gather, warp = 32 consecutive z voxels of one (i, j) column (lanes along
// z): a cone view's detector COLUMN window depends on (x, y) only, so the warp walks one
// column range together, each lane its own row window; the projections (transposed to
// pt[a][iu][iv]) and the ray table (same order) are read along detector columns, i.e.
// coalesced across the lanes.  Per voxel the contributions are added in the reference's
// scatter order (view, row, column) -- the lane's row loop is inside the column loop here,
// so the order is kept by iterating rows outermost per lane.
#ifndef CTK_SID_MINB
#define CTK_SID_MINB 6  // 113 -> 80 regs (80 B spill): 58.8 -> 55.4 ms at 256^3/180 (5: 57.4, 8: 56.6)
#endif
// zonly: only the z-dominant cone rays (the f32 slab model's complement), accumulated into vol
template <class T>
__global__ void __launch_bounds__(128, CTK_SID_MINB) k_siddon_atb(KGeom g, const double* __restrict__ rayinv,
                                                    const T* __restrict__ pt, T* __restrict__ vol, int kblocks,
                                                    int zonly) {
    const long wid = long(blockIdx.x) * blockDim.y + threadIdx.y;
    const long ncol = long(g.nx) * g.ny;
    if (wid >= ncol * kblocks) return;
    const int kb = int(wid / ncol) * 32;
    const long col = wid % ncol;
    const int idx3[3] = {int(col % g.nx), int(col / g.nx), kb + int(threadIdx.x)};
    const bool live = idx3[2] < g.nz;
    const int n3[3] = {g.nx, g.ny, g.nz};
    const double h = g.h;
    const double lo3[3] = {(idx3[0] - 0.5 * g.nx) * h, (idx3[1] - 0.5 * g.ny) * h, (idx3[2] - 0.5 * g.nz) * h};
    double plo[3], phi[3];  // the voxel's six crossing planes, (q - n/2) h exactly as s_alpha forms them
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        plo[ax] = (idx3[ax] - 0.5 * n3[ax]) * h;
        phi[ax] = (idx3[ax] + 1 - 0.5 * n3[ax]) * h;
    }
    const size_t frame = size_t(g.nu) * g.nv;
    const bool cone = g.mode == CTK_CONE3D;
    T acc = 0;
    for (int a = 0; a < g.na && live; ++a) {
        const double2 cs = g.ctst[a];
        int iu0 = 0, iu1 = g.nu - 1, iv0 = 0, iv1 = g.nv - 1;
        if (!s_window(g, cs.x, cs.y, lo3, h, iu0, iu1, iv0, iv1)) {
            iu0 = 0; iu1 = g.nu - 1; iv0 = 0; iv1 = g.nv - 1;
        }
        const double sx = g.dso * cs.x, sy = g.dso * cs.y;  // cone: every ray starts at the source
        const T* fa = pt + size_t(a) * frame;
        const double* ra = rayinv + 3 * size_t(a) * frame;
        if (cone) {
            // every ray of the view starts at the source: the plane offsets (plane - o) are
            // per (voxel, view), the same subtractions the general path does per candidate
            const double o3[3] = {sx, sy, 0.0};
            double dlo[3], dhi[3];
            bool flat[3];
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                dlo[ax] = plo[ax] - o3[ax];
                dhi[ax] = phi[ax] - o3[ax];
                flat[ax] = s_slab(o3[ax], n3[ax], h) == idx3[ax];  // a ray with d_ax == 0 stays in o's slab
            }
            for (int iv = iv0; iv <= iv1; ++iv)
                for (int iu = iu0; iu <= iu1; ++iu) {
                    const size_t q = size_t(iu) * g.nv + iv;  // [a][iu][iv]
                    const T value = __ldg(fa + q);
                    if (value == T(0)) continue;
                    if (zonly && !(fabs((iv - 0.5 * (g.nv - 1)) * g.du) > g.colstep[a * g.nu + iu].y)) continue;
                    const double inv[3] = {__ldg(ra + 3 * q), __ldg(ra + 3 * q + 1), __ldg(ra + 3 * q + 2)};
                    double lo = -DBL_MAX, hi = DBL_MAX;
                    bool miss = false;
#pragma unroll
                    for (int ax = 0; ax < 3; ++ax) {
                        if (inv[ax] == 0.0) {
                            miss |= !flat[ax];
                            continue;
                        }
                        const double a0 = dlo[ax] * inv[ax];
                        const double a1 = dhi[ax] * inv[ax];
                        lo = fmax(lo, fmin(a0, a1));
                        hi = fmin(hi, fmax(a0, a1));
                    }
                    if (miss || !(hi > lo)) continue;
                    acc += T(hi - lo) * value;
                }
            continue;
        }
        for (int iv = iv0; iv <= iv1; ++iv)
            for (int iu = iu0; iu <= iu1; ++iu) {
                const size_t q = size_t(iu) * g.nv + iv;  // [a][iu][iv]
                const T value = __ldg(fa + q);
                if (value == T(0)) continue;
                const double inv[3] = {__ldg(ra + 3 * q), __ldg(ra + 3 * q + 1), __ldg(ra + 3 * q + 2)};
                double o[3];
                if (cone) {
                    o[0] = sx; o[1] = sy; o[2] = 0.0;
                } else {  // make_ray's parallel origin, operation for operation
                    const double u = (iu - 0.5 * (g.nu - 1)) * g.du;
                    const double v = (iv - 0.5 * (g.nv - 1)) * g.du;
                    const double cx = -g.dod * cs.x, cy = -g.dod * cs.y, cz = 0.0;
                    o[0] = cx - u * cs.y; o[1] = cy + u * cs.x; o[2] = cz + v;
                }
                double lo = -DBL_MAX, hi = DBL_MAX;
                bool miss = false;
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) {
                    if (inv[ax] == 0.0) {  // d_ax == 0
                        if (s_slab(o[ax], n3[ax], h) != idx3[ax]) miss = true;
                        continue;
                    }
                    const double a0 = (plo[ax] - o[ax]) * inv[ax];
                    const double a1 = (phi[ax] - o[ax]) * inv[ax];
                    lo = fmax(lo, fmin(a0, a1));
                    hi = fmin(hi, fmax(a0, a1));
                }
                if (miss || !(hi > lo)) continue;
                acc += T(hi - lo) * value;
            }
    }
    if (live) {
        T* o = vol + size_t(idx3[0]) + size_t(g.nx) * (size_t(idx3[1]) + size_t(g.ny) * idx3[2]);
        *o = zonly ? *o + acc : acc;
    }
}

// y[a][iv][iu] -> pt[a][iu][iv]
template <class T>
__global__ void k_siddon_transpose(int nu, int nv, const T* __restrict__ y, T* __restrict__ pt) {
    __shared__ T tile[32][33];
    const int a = blockIdx.z, u0 = blockIdx.x * 32, v0 = blockIdx.y * 32;
    const size_t frame = size_t(nu) * nv;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int iu = u0 + threadIdx.x, iv = v0 + r;
        tile[r][threadIdx.x] = (iu < nu && iv < nv) ? y[a * frame + size_t(iv) * nu + iu] : T(0);
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int iu = u0 + r, iv = v0 + threadIdx.x;
        if (iu < nu && iv < nv) pt[a * frame + size_t(iu) * nv + iv] = tile[threadIdx.x][r];
    }
}

}  // namespace

template <class T>
void siddon_ax(const Geometry& g, const T* x, T* y, cudaStream_t s) {
    dim3 blk(32, 4), grd((g.nu + 31) / 32, (g.nv + 3) / 4, g.na);
    k_siddon_ax<T><<<grd, blk, 0, s>>>(g.kgeom(), x, y, 0);
    after_launch("k_siddon_ax");
}

void siddon_ax_zrays_f32(const Geometry& g, const float* x, float* y, cudaStream_t s) {
    dim3 blk(32, 4), grd((g.nu + 31) / 32, (g.nv + 3) / 4, g.na);
    k_siddon_ax<float><<<grd, blk, 0, s>>>(g.kgeom(), x, y, 1);
    after_launch("k_siddon_ax_zrays");
}

template <class T>
void siddon_atb_impl(Geometry& g, const T* y, T* x, cudaStream_t s, int zonly) {
    const size_t nrays = g.range();
    if (g.d_rayinv.ensure(3 * nrays * sizeof(double)) || !g.rayinv_ready) {
        dim3 blk(32, 4), grd((g.nu + 31) / 32, (g.nv + 3) / 4, g.na);
        k_siddon_rayinv<<<grd, blk, 0, s>>>(g.kgeom(), g.d_rayinv.as<double>());
        after_launch("k_siddon_rayinv");
        g.rayinv_ready = true;
    }
    g.proj_t.ensure(nrays * sizeof(T));
    {
        dim3 blk(32, 8), grd((g.nu + 31) / 32, (g.nv + 31) / 32, g.na);
        k_siddon_transpose<T><<<grd, blk, 0, s>>>(g.nu, g.nv, y, g.proj_t.as<T>());
        after_launch("k_siddon_transpose");
    }
    const int kblocks = (g.nz + 31) / 32;
    const long warps = long(g.nx) * g.ny * kblocks;
    dim3 blk(32, 4);
    k_siddon_atb<T><<<unsigned((warps + 3) / 4), blk, 0, s>>>(g.kgeom(), g.d_rayinv.as<double>(), g.proj_t.as<T>(), x,
                                                            kblocks, zonly);
    after_launch(zonly ? "k_siddon_atb_zrays" : "k_siddon_atb");
}

template <class T>
void siddon_atb(Geometry& g, const T* y, T* x, cudaStream_t s) {
    siddon_atb_impl<T>(g, y, x, s, 0);
}

// the f32 slab-model transpose (bp_f32.cu) leaves the z-dominant rays to this exact gather;
// it overwrites proj_t, so it runs after the plane passes
void siddon_atb_zrays_f32(Geometry& g, const float* y, float* x, cudaStream_t s) { siddon_atb_impl<float>(g, y, x, s, 1); }

template void siddon_ax<float>(const Geometry&, const float*, float*, cudaStream_t);
template void siddon_ax<double>(const Geometry&, const double*, double*, cudaStream_t);
template void siddon_atb<float>(Geometry&, const float*, float*, cudaStream_t);
template void siddon_atb<double>(Geometry&, const double*, double*, cudaStream_t);

}  // namespace ctkb
