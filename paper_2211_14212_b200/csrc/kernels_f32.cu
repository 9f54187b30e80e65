// sm_100a performance kernels for T = float: Joseph forward projection (Ax) and its
// exact transpose / the voxel-driven backprojection (A^T b).
//
// Ray model (separable restatement of make_ray + plan_walk, projector.hpp:29-91).  For a
// view a and detector column iu, the unnormalised ray d = P - S has horizontal part
// (dx, dy) independent of the detector row.  Rays whose dominant axis A is x or y
// (|d_A| >= |dz|) walk the slices s of A; in slice s the ray sits at
//     fh(s) = fh0 + s*fhd                   (in-plane horizontal index: y if A=x, x if A=y)
//     fz(s) = vd(iv) * (g0 + s*gd) + cz     (z index; vd = detector row coordinate)
// with {fh0, fhd, g0, gd} a per-(view, column) f32 table computed in fp64 on the host,
// and path length per slice step = h*|d|/|d_A| (= h/|dir_A|, projector.hpp:77).  Both
// the forward and the transpose evaluate exactly these f32 expressions, so the matched
// A^T b is the exact transpose of this Ax up to fp32 rounding of the products.  Rays with
// a dominant z component (steep cone rows) take a generic per-ray path.
//
// Layouts in HBM (f32):
//   qx[i][k+1][j+1]  bilinear quads (16 B) of each x-slice plane      (x-dominant rays)
//   qy[j][k+1][i+1]  bilinear quads (16 B) of each y-slice plane      (y-dominant rays)
// so that a warp of 32 consecutive detector columns reads 32 consecutive quads per
// sample: one 16-byte load, no bounds checks (zero padding is in the quads).
//   proj_t[a][iu][iv] detector columns contiguous (gathers read consecutive rows).
#include <cfloat>
#include <cstdlib>

#include "ctk_internal.h"
#include "reduce.cuh"

namespace ctkb {
namespace {

constexpr int FWD_BX = 32, FWD_BY = 8;  // rays per forward block: 32 columns x 8 rows

__device__ __forceinline__ double row_coord(const KGeom& g, int iv) { return (iv - 0.5 * (g.nv - 1)) * g.du; }

// path length per slice step of ray (column c, row coordinate v)
__device__ __forceinline__ float ray_step(const KGeom& g, double2 cs, double v) {
    if (g.mode == CTK_CONE3D) {
        const double av = fabs(v);
        const double dom = av > cs.y ? av : cs.y;
        return float(g.h * sqrt(cs.x + v * v) / dom);
    }
    return float(g.h / cs.y);
}

__device__ __forceinline__ bool is_zray(const KGeom& g, double2 cs, double v) {
    return g.mode == CTK_CONE3D && fabs(v) > cs.y;
}

__device__ __forceinline__ void clip_affine(double f0, double fd, double lo, double hi, int& s0, int& s1) {
    if (fd == 0.0) {
        if (!(f0 > lo - 1.0 && f0 < hi + 1.0)) { s0 = 1; s1 = 0; }
        return;
    }
    double a = (lo - f0) / fd, b = (hi - f0) / fd;
    if (a > b) { const double t = a; a = b; b = t; }
    if (a > 2e9 || b < -2e9) { s0 = 1; s1 = 0; return; }
    s0 = max(s0, int(floor(fmax(a, -2e9))) - 1);
    s1 = min(s1, int(ceil(fmin(b, 2e9))) + 1);
}

// ---- generic walk (z-dominant rays): plan_walk in fp64, positions in f32 ----------------
struct WalkF {
    int axis, ns, nb, nc;
    float fb0, fbd, fc0, fcd, step;
    int sa, sb, sc;
};

__device__ void walk_generic(const KGeom& g, double ct, double st, int iu, int iv, WalkF& w) {
    const double u = (iu - 0.5 * (g.nu - 1)) * g.du;
    const double v = (iv - 0.5 * (g.nv - 1)) * g.du;
    double o[3], d[3];
    const double px = -g.dod * ct - u * st, py = -g.dod * st + u * ct, pz = v;
    if (g.mode == CTK_CONE3D) {
        o[0] = g.dso * ct; o[1] = g.dso * st; o[2] = 0.0;
        d[0] = px - o[0]; d[1] = py - o[1]; d[2] = pz;
        const double n = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        d[0] /= n; d[1] /= n; d[2] /= n;
    } else {
        o[0] = px; o[1] = py; o[2] = pz;
        d[0] = -ct; d[1] = -st; d[2] = 0.0;
    }
    const double ad0 = fabs(d[0]), ad1 = fabs(d[1]), ad2 = fabs(d[2]);
    int axis = 0;
    double adm = ad0;
    if (ad1 > adm) { axis = 1; adm = ad1; }
    if (ad2 > adm) { axis = 2; adm = ad2; }
    const int n3[3] = {g.nx, g.ny, g.nz};
    const int s3[3] = {1, g.nx, g.nx * g.ny};
    const int b = axis == 2 ? 0 : axis + 1, c = axis == 0 ? 2 : axis - 1;
    const double h = g.h;
    const double t0 = ((0 - 0.5 * (n3[axis] - 1)) * h - o[axis]) / d[axis];
    const double dt = h / d[axis];
    w.axis = axis;
    w.ns = n3[axis];
    w.nb = n3[b];
    w.nc = n3[c];
    w.sa = s3[axis];
    w.sb = s3[b];
    w.sc = s3[c];
    w.step = float(h / adm);
    w.fb0 = float((o[b] + t0 * d[b]) / h + 0.5 * (n3[b] - 1));
    w.fbd = float(dt * d[b] / h);
    w.fc0 = float((o[c] + t0 * d[c]) / h + 0.5 * (n3[c] - 1));
    w.fcd = float(dt * d[c] / h);
}

__device__ float march_generic(const KGeom& g, const WalkF& w, const float* __restrict__ vol) {
    int s0 = 0, s1 = w.ns - 1;
    clip_affine(w.fb0, w.fbd, -1.0, w.nb, s0, s1);
    clip_affine(w.fc0, w.fcd, -1.0, w.nc, s0, s1);
    float acc = 0.f;
    for (int s = s0; s <= s1; ++s) {
        const float fb = fmaf(float(s), w.fbd, w.fb0);
        const float fc = fmaf(float(s), w.fcd, w.fc0);
        const float fib = floorf(fb), fic = floorf(fc);
        const int ib = int(fib), ic = int(fic);
        const float tb = fb - fib, tc = fc - fic;
        const float* p = vol + size_t(s) * w.sa;
        const bool b0 = ib >= 0 && ib < w.nb, b1 = ib + 1 >= 0 && ib + 1 < w.nb;
        const bool c0 = ic >= 0 && ic < w.nc, c1 = ic + 1 >= 0 && ic + 1 < w.nc;
        const float v00 = (b0 && c0) ? __ldg(p + ib * w.sb + ic * w.sc) : 0.f;
        const float v10 = (b1 && c0) ? __ldg(p + (ib + 1) * w.sb + ic * w.sc) : 0.f;
        const float v01 = (b0 && c1) ? __ldg(p + ib * w.sb + (ic + 1) * w.sc) : 0.f;
        const float v11 = (b1 && c1) ? __ldg(p + (ib + 1) * w.sb + (ic + 1) * w.sc) : 0.f;
        const float a0 = fmaf(tb, v10 - v00, v00);
        const float a1 = fmaf(tb, v11 - v01, v01);
        acc += fmaf(tc, a1 - a0, a0);
    }
    return w.step * acc;
}
// ---- quad relayout: x[i + nx(j + ny k)] -> bilinear quads per slice plane -------------
// qx[i][k+1][j+1] = (v(i,j,k), v(i,j+1,k), v(i,j,k+1), v(i,j+1,k+1))   x-dominant rays
// qy[j][k+1][i+1] = (v(i,j,k), v(i+1,j,k), v(i,j,k+1), v(i+1,j,k+1))   y-dominant rays
// for in-plane indices h in [-1, nh-1] and k in [-1, nz-1]; taps outside the volume are 0
// (Joseph's zero padding, projector.hpp:108).  One 16-byte load per bilinear sample.
__device__ __forceinline__ float vox(const float* __restrict__ x, int nx, int ny, int nz, int i, int j, int k) {
    return (i >= 0 && i < nx && j >= 0 && j < ny && k >= 0 && k < nz)
               ? __ldg(x + size_t(i) + size_t(nx) * (size_t(j) + size_t(ny) * k))
               : 0.f;
}

__global__ void k_quads_y(int nx, int ny, int nz, const float* __restrict__ x, float4* __restrict__ qy) {
    const int io = blockIdx.x * blockDim.x + threadIdx.x;  // i + 1
    const int ko = blockIdx.y;                             // k + 1
    const int j = blockIdx.z;
    if (io > nx) return;
    const int i = io - 1, k = ko - 1;
    const size_t pitch = size_t(nx) + 1, plane = pitch * (size_t(nz) + 1);
    qy[size_t(j) * plane + size_t(ko) * pitch + io] =
        make_float4(vox(x, nx, ny, nz, i, j, k), vox(x, nx, ny, nz, i + 1, j, k), vox(x, nx, ny, nz, i, j, k + 1),
                    vox(x, nx, ny, nz, i + 1, j, k + 1));
}

// 32(i) x 33(j) x 2(k) tile through shared memory so both the reads (along i) and the
// quad writes (along j) are coalesced
__global__ void k_quads_x(int nx, int ny, int nz, const float* __restrict__ x, float4* __restrict__ qx) {
    __shared__ float tile[2][33][33];
    const int i0 = blockIdx.x * 32, jo0 = blockIdx.y * 32, ko = blockIdx.z;
    const int k = ko - 1;
    for (int r = threadIdx.y; r < 2 * 33; r += blockDim.y) {
        const int kz = r / 33, jj = r % 33;
        tile[kz][jj][threadIdx.x] = vox(x, nx, ny, nz, i0 + threadIdx.x, jo0 - 1 + jj, k + kz);
    }
    __syncthreads();
    const size_t pitch = size_t(ny) + 1, plane = pitch * (size_t(nz) + 1);
    const int jo = jo0 + threadIdx.x;  // j + 1
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int i = i0 + r;
        if (i < nx && jo <= ny) {
            const int jj = threadIdx.x;  // tile row of j = jo - 1
            qx[size_t(i) * plane + size_t(ko) * pitch + jo] =
                make_float4(tile[0][jj][r], tile[0][jj + 1][r], tile[1][jj][r], tile[1][jj + 1][r]);
        }
    }
}

// floor without the conversion pipe: t = (f - 0.5) + 1.5*2^23 rounds to an integer n with
// n = floor(f) except at exact integers, where n may be f - 1 with frac 1.0 -- the same
// bilinear weights (1 on tap f).  Valid for |f| < 2^22.
__device__ __forceinline__ void split(float f, int& i, float& frac) {
    const float M = 12582912.0f;
    const float t = __fadd_rn(__fadd_rn(f, -0.5f), M);
    const float fi = __fadd_rn(t, -M);
    i = __float_as_int(t) - __float_as_int(M);
    frac = __fadd_rn(f, -fi);
}

// ---- forward projection ----------------------------------------------------------------
// RESID=false: y[a][iv][iu] = A x.   RESID=true: per-block partial of sum (Ax - b)^2.
template <bool RESID>
__global__ void __launch_bounds__(FWD_BX * FWD_BY)
k_ax_f32(KGeom g, const float4* __restrict__ qx, const float4* __restrict__ qy, const float* __restrict__ xs,
         float* __restrict__ y, const float* __restrict__ b, double* __restrict__ partials) {
    const int iu = blockIdx.x * FWD_BX + threadIdx.x;
    const int iv = blockIdx.y * FWD_BY + threadIdx.y;
    const int a = blockIdx.z;
    float out = 0.f;
    const bool live = iu < g.nu && iv < g.nv;
    if (live) {
        const int c = a * g.nu + iu;
        const double2 cs = g.colstep[c];
        const double v = row_coord(g, iv);
        if (g.has_zrays && is_zray(g, cs, v)) {
            const double2 tr = g.ctst[a];
            WalkF w;
            walk_generic(g, tr.x, tr.y, iu, iv, w);
            out = march_generic(g, w, xs);
        } else {
            const float4 cd = g.col[c];
            const int A = g.colaxis[c];
            const int nh = A ? g.nx : g.ny;
            const int ns = A ? g.ny : g.nx;
            const int pitch = nh + 1;
            const int plane = pitch * (g.nz + 1);
            const float4* base = (A ? qy : qx) + pitch + 1;  // quad of (h, z) at base[z*pitch + h]
            const float vd = float(v);
            const float czf = 0.5f * float(g.nz - 1);
            int s0 = 0, s1 = ns - 1;
            clip_affine(cd.x, cd.y, -1.0, nh, s0, s1);
            clip_affine(double(vd) * cd.z + czf, double(vd) * cd.w, -1.0, g.nz, s0, s1);
            float acc = 0.f;
            const unsigned unh = unsigned(nh), unz = unsigned(g.nz);
#pragma unroll 4
            for (int s = s0; s <= s1; ++s) {
                const float fs = float(s);
                const float fh = fmaf(fs, cd.y, cd.x);
                const float gs = fmaf(fs, cd.w, cd.z);
                const float fz = fmaf(vd, gs, czf);
                int ih, iz;
                float th, tz;
                split(fh, ih, th);
                split(fz, iz, tz);
                // sample inside the padded plane <=> some tap inside the volume
                const bool in = unsigned(ih + 1) <= unh && unsigned(iz + 1) <= unz;
                const int off = in ? s * plane + iz * pitch + ih : -pitch - 1;  // -pitch-1: quad (-1,-1), in bounds
                const float4 q = __ldg(base + off);
                const float a0 = fmaf(th, q.y - q.x, q.x);
                const float a1 = fmaf(th, q.w - q.z, q.z);
                const float smp = fmaf(tz, a1 - a0, a0);
                acc += in ? smp : 0.f;
            }
            out = ray_step(g, cs, v) * acc;
        }
    }
    const size_t o = size_t(a) * g.nu * g.nv + size_t(iv) * g.nu + iu;
    if (!RESID) {
        if (live) y[o] = out;
    } else {
        double r = 0.0;
        if (live) {
            const double d = double(out) - double(__ldg(b + o));
            r = d * d;
        }
        r = block_sum(r);
        if (threadIdx.x == 0 && threadIdx.y == 0)
            partials[(size_t(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = r;
    }
}

// ---- projection transpose for the gathers: pt[a][iu][iv] = (step?) * y[a][iv][iu] ------
template <bool SCALE>
__global__ void k_proj_transpose(KGeom g, const float* __restrict__ y, float* __restrict__ pt) {
    __shared__ float tile[32][33];
    const int a = blockIdx.z;
    const int u0 = blockIdx.x * 32, v0 = blockIdx.y * 32;
    const float* fr = y + size_t(a) * g.nu * g.nv;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int iu = u0 + threadIdx.x, iv = v0 + r;
        tile[r][threadIdx.x] = (iu < g.nu && iv < g.nv) ? __ldg(fr + size_t(iv) * g.nu + iu) : 0.f;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int iu = u0 + r, iv = v0 + threadIdx.x;
        if (iu < g.nu && iv < g.nv) {
            float val = tile[threadIdx.x][r];
            const int c = a * g.nu + iu;
            if (SCALE) val *= ray_step(g, g.colstep[c], row_coord(g, iv));
            pt[size_t(c) * g.nv + iv] = val;
        }
    }
}

// horizontal detector coordinate (continuous pixel index) of the point (x, y)
__device__ __forceinline__ double proj_u(const KGeom& g, double ct, double st, double x, double y, bool& ok) {
    ok = true;
    if (g.mode == CTK_CONE3D) {
        const double sx = g.dso * ct, sy = g.dso * st;
        const double rx = x - sx, ry = y - sy;
        const double depth = -(rx * ct + ry * st);
        if (!(depth > 1e-9 * g.dso)) { ok = false; return 0.0; }
        const double t = (g.dso + g.dod) / depth;
        return (-(sx + t * rx) * st + (sy + t * ry) * ct) / g.du + 0.5 * (g.nu - 1);
    }
    return (-x * st + y * ct) / g.du + 0.5 * (g.nu - 1);
}

// ---- matched A^T b, plane-driven ------------------------------------------------------
// Pass CLASS (0: x-dominant columns, planes x = s, rows p = y; 1: y-dominant columns,
// planes y = s, rows p = x).  A CTA owns one plane s, BP_PB rows [p0, p0+BP_PB) and a band
// of BP_KB slices [k0, k0+BP_KB) along z, and loops over all views.  Per view:
//  phase 1  one thread per candidate detector column iu marches its detector rows iv
//           (exactly the forward's f32 fz = fmaf(vd, fmaf(s, gd, g0), cz); 16-byte column
//           loads) and accumulates the transposed z-interpolation Z[k][e] = sum wz*(step*y)
//           in shared memory; it registers itself in the (at most two) rows its in-plane
//           stencil touches;
//  phase 2  thread p owns row p (BP_KB accumulators in registers) and adds wh * Z[:][e] of
//           the columns registered in its row, sorted by column -> deterministic order.
// Z[k][e] has row stride BP_PB: phase-1 lanes (consecutive e) hit distinct banks whatever
// their k, phase-2 lanes (consecutive rows -> consecutive e) likewise.
constexpr int BP_PB = 256, BP_KB = 32, BP_SL = 8;

template <int CLASS>
__global__ void __launch_bounds__(BP_PB)
k_atb_plane_f32(KGeom g, const float* __restrict__ pt, float* __restrict__ x, int ptiles) {
    extern __shared__ __align__(16) float sm[];
    float* Z = sm;                                              // [BP_KB][BP_PB]
    int* lists = reinterpret_cast<int*>(Z + BP_KB * BP_PB);     // [BP_PB][BP_SL]
    int* cnt = lists + BP_PB * BP_SL;                           // [BP_PB]
    float* eth = reinterpret_cast<float*>(cnt + BP_PB);         // [BP_PB]
    float* vdtab = eth + BP_PB;                                 // [nv]
    __shared__ int s_iu0, s_iu1;

    const int t = threadIdx.x;
    const int s = blockIdx.y;
    const int ptile = blockIdx.x % ptiles, kband = blockIdx.x / ptiles;
    const int p0 = ptile * BP_PB, k0 = kband * BP_KB;
    const int nh = CLASS ? g.nx : g.ny;
    const int p = p0 + t;
    for (int q = t; q < g.nv; q += BP_PB) vdtab[q] = float(row_coord(g, q));
    const float czf = 0.5f * float(g.nz - 1);
    const float cvf = 0.5f * float(g.nv - 1);
    const float invdu = float(1.0 / g.du);
    const float fs = float(s);
    const double h = g.h;
    const bool vec4 = (g.nv & 3) == 0;
    // world coordinates of the plane and of the tile's row segment ends
    const double plane_c = (s - 0.5 * ((CLASS ? g.ny : g.nx) - 1)) * h;
    const double r_lo = (p0 - 1.5 - 0.5 * (nh - 1)) * h, r_hi = (p0 + BP_PB + 0.5 - 0.5 * (nh - 1)) * h;

    float acc[BP_KB];
#pragma unroll
    for (int m = 0; m < BP_KB; ++m) acc[m] = 0.f;

    for (int a = 0; a < g.na; ++a) {
        if (t == 0) {
            const double2 tr = g.ctst[a];
            bool ok1, ok2;
            const double u1 = CLASS ? proj_u(g, tr.x, tr.y, r_lo, plane_c, ok1) : proj_u(g, tr.x, tr.y, plane_c, r_lo, ok1);
            const double u2 = CLASS ? proj_u(g, tr.x, tr.y, r_hi, plane_c, ok2) : proj_u(g, tr.x, tr.y, plane_c, r_hi, ok2);
            int i0 = 0, i1 = g.nu - 1;
            if (ok1 && ok2) {
                i0 = max(i0, int(floor(fmax(fmin(u1, u2), -1e9))) - 1);
                i1 = min(i1, int(ceil(fmin(fmax(u1, u2), 1e9))) + 1);
            }
            s_iu0 = i0;
            s_iu1 = i1;
        }
        __syncthreads();
        const int iu0 = s_iu0, iu1 = s_iu1;
        __syncthreads();  // s_iu* is rewritten for the next view
        for (int cbase = iu0; cbase <= iu1; cbase += BP_PB) {
            // ---- phase 1 ----
            cnt[t] = 0;
            __syncthreads();
            const int iu = cbase + t;
            if (iu <= iu1) {
                const int c = a * g.nu + iu;
                if (g.colaxis[c] == CLASS) {
                    const float4 cd = g.col[c];
                    const float fh = fmaf(fs, cd.y, cd.x);
                    const float fih = floorf(fh);
                    const int ih = int(fih);
                    const float th = fh - fih;
                    if (ih + 1 >= p0 && ih <= p0 + BP_PB - 1 && ih + 1 >= 0 && ih < nh) {
#pragma unroll
                        for (int m = 0; m < BP_KB; ++m) Z[m * BP_PB + t] = 0.f;
                        const float gs = fmaf(fs, cd.w, cd.z);
                        int v0 = 0, v1 = g.nv - 1;
                        if (gs > 0.f) {
                            const float rg = invdu / gs;
                            v0 = max(v0, int(floorf(fmaf(float(k0) - 1.f - czf, rg, cvf))) - 1);
                            v1 = min(v1, int(ceilf(fmaf(float(k0 + BP_KB) - czf, rg, cvf))) + 1);
                        }
                        const double dA = g.colstep[c].y;
                        const float* pc = pt + size_t(c) * g.nv;
                        auto add = [&](int iv, float yv) {
                            if (g.has_zrays && fabs(row_coord(g, iv)) > dA) return;
                            const float fz = fmaf(vdtab[iv], gs, czf);
                            const float fiz = floorf(fz);
                            const int kk = int(fiz) - k0;
                            const float tz = fz - fiz;
                            if (kk >= 0 && kk < BP_KB) Z[kk * BP_PB + t] = fmaf(1.f - tz, yv, Z[kk * BP_PB + t]);
                            if (kk + 1 >= 0 && kk + 1 < BP_KB) Z[(kk + 1) * BP_PB + t] = fmaf(tz, yv, Z[(kk + 1) * BP_PB + t]);
                        };
                        if (vec4) {
                            for (int b4 = v0 & ~3; b4 <= v1; b4 += 4) {
                                const float4 y4 = __ldg(reinterpret_cast<const float4*>(pc + b4));
                                if (b4 >= v0) add(b4, y4.x);
                                if (b4 + 1 >= v0 && b4 + 1 <= v1) add(b4 + 1, y4.y);
                                if (b4 + 2 >= v0 && b4 + 2 <= v1) add(b4 + 2, y4.z);
                                if (b4 + 3 <= v1) add(b4 + 3, y4.w);
                            }
                        } else {
                            for (int iv = v0; iv <= v1; ++iv) add(iv, __ldg(pc + iv));
                        }
                        eth[t] = th;
                        if (ih >= p0) {
                            const int sl = atomicAdd(&cnt[ih - p0], 1);
                            if (sl < BP_SL) lists[(ih - p0) * BP_SL + sl] = (t << 1);
                        }
                        if (ih + 1 <= p0 + BP_PB - 1 && th != 0.f) {
                            const int sl = atomicAdd(&cnt[ih + 1 - p0], 1);
                            if (sl < BP_SL) lists[(ih + 1 - p0) * BP_SL + sl] = (t << 1) | 1;
                        }
                    }
                }
            }
            __syncthreads();
            // ---- phase 2: row p gathers its registered columns in column order ----
            const int n = cnt[t];
            if (n > 0 && p < nh) {
                if (n <= BP_SL) {
                    int lst[BP_SL];
#pragma unroll
                    for (int q = 0; q < BP_SL; ++q) lst[q] = q < n ? lists[t * BP_SL + q] : 0x7fffffff;
#pragma unroll
                    for (int i = 1; i < BP_SL; ++i)
#pragma unroll
                        for (int j = BP_SL - 1; j >= i; --j)
                            if (lst[j - 1] > lst[j]) { const int tmp = lst[j]; lst[j] = lst[j - 1]; lst[j - 1] = tmp; }
#pragma unroll
                    for (int q = 0; q < BP_SL; ++q) {
                        if (q >= n) break;
                        const int e = lst[q] >> 1;
                        const float th = eth[e];
                        const float wh = (lst[q] & 1) ? th : 1.f - th;
#pragma unroll
                        for (int m = 0; m < BP_KB; ++m) acc[m] = fmaf(wh, Z[m * BP_PB + e], acc[m]);
                    }
                } else {
                    // overflow (very fine detector sampling): scan every column of the chunk in order
                    for (int e = 0; e < BP_PB && cbase + e <= iu1; ++e) {
                        const int c = a * g.nu + cbase + e;
                        if (g.colaxis[c] != CLASS) continue;
                        const float4 cd = g.col[c];
                        const float fh = fmaf(fs, cd.y, cd.x);
                        const float fih = floorf(fh);
                        const int ih = int(fih);
                        const float th = fh - fih;
                        float wh;
                        if (ih == p) wh = 1.f - th;
                        else if (ih + 1 == p && th != 0.f) wh = th;
                        else continue;
#pragma unroll
                        for (int m = 0; m < BP_KB; ++m) acc[m] = fmaf(wh, Z[m * BP_PB + e], acc[m]);
                    }
                }
            }
            __syncthreads();
        }
    }
    if (p < nh) {
#pragma unroll
        for (int m = 0; m < BP_KB; ++m) {
            const int k = k0 + m;
            if (k >= g.nz) break;
            const size_t o = CLASS ? size_t(p) + size_t(g.nx) * (size_t(s) + size_t(g.ny) * k)
                                   : size_t(s) + size_t(g.nx) * (size_t(p) + size_t(g.ny) * k);
            if (CLASS == 0) x[o] = acc[m];
            else x[o] += acc[m];
        }
    }
}

__global__ void k_atb_matched_zrays_f32(KGeom g, const float* __restrict__ pt, float* __restrict__ x) {
    const size_t nvox = size_t(g.nx) * g.ny * g.nz;
    const size_t id = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (id >= nvox) return;
    const int i = int(id % g.nx), j = int((id / g.nx) % g.ny), k = int(id / (size_t(g.nx) * g.ny));
    const double h = g.h;
    const double xc = (i - 0.5 * (g.nx - 1)) * h, yc = (j - 0.5 * (g.ny - 1)) * h, zc = (k - 0.5 * (g.nz - 1)) * h;
    float acc = 0.f;
    for (int a = 0; a < g.na; ++a) {
        const double2 tr = g.ctst[a];
        const double sx = g.dso * tr.x, sy = g.dso * tr.y;
        double umin = DBL_MAX, umax = -DBL_MAX, vmin = DBL_MAX, vmax = -DBL_MAX;
        bool all = false;
        for (int q = 0; q < 8; ++q) {
            const double px = xc + ((q & 1) ? h : -h), py = yc + ((q & 2) ? h : -h), pz = zc + ((q & 4) ? h : -h);
            const double rx = px - sx, ry = py - sy;
            const double depth = -(rx * tr.x + ry * tr.y);
            if (!(depth > 1e-9 * g.dso)) { all = true; break; }
            const double t = (g.dso + g.dod) / depth;
            const double fu = (-(sx + t * rx) * tr.y + (sy + t * ry) * tr.x) / g.du + 0.5 * (g.nu - 1);
            const double fv = t * pz / g.du + 0.5 * (g.nv - 1);
            umin = fmin(umin, fu); umax = fmax(umax, fu);
            vmin = fmin(vmin, fv); vmax = fmax(vmax, fv);
        }
        int iu0 = 0, iu1 = g.nu - 1, iv0 = 0, iv1 = g.nv - 1;
        if (!all) {
            iu0 = max(iu0, int(floor(fmax(umin, -1e9))) - 1);
            iu1 = min(iu1, int(ceil(fmin(umax, 1e9))) + 1);
            iv0 = max(iv0, int(floor(fmax(vmin, -1e9))) - 1);
            iv1 = min(iv1, int(ceil(fmin(vmax, 1e9))) + 1);
        }
        for (int iv = iv0; iv <= iv1; ++iv) {
            const double v = row_coord(g, iv);
            for (int iu = iu0; iu <= iu1; ++iu) {
                const int c = a * g.nu + iu;
                if (!is_zray(g, g.colstep[c], v)) continue;
                WalkF w;
                walk_generic(g, tr.x, tr.y, iu, iv, w);
                // axis is z: slice k, b = x (i), c = y (j)
                const float fs = float(k);
                const float fb = fmaf(fs, w.fbd, w.fb0), fc = fmaf(fs, w.fcd, w.fc0);
                const float fib = floorf(fb), fic = floorf(fc);
                const int ib = int(fib), ic = int(fic);
                const float tb = fb - fib, tc = fc - fic;
                float wb, wc;
                if (i == ib) wb = 1.f - tb; else if (i == ib + 1) wb = tb; else continue;
                if (j == ic) wc = 1.f - tc; else if (j == ic + 1) wc = tc; else continue;
                acc = fmaf(wb * wc, __ldg(pt + size_t(c) * g.nv + iv), acc);
            }
        }
    }
    x[id] += acc;
}

// ---- voxel-driven A^T b (projector.hpp:204-279), warp per column as above --------------
template <int KZ>
__global__ void __launch_bounds__(128)
k_atb_voxel_f32(KGeom g, const float* __restrict__ pt, float* __restrict__ x, int kblocks) {
    const int lane = threadIdx.x;
    const long wid = long(blockIdx.x) * blockDim.y + threadIdx.y;
    const long ncol = long(g.nx) * g.ny;
    if (wid >= ncol * kblocks) return;
    const int kb = int(wid / ncol) * 32 * KZ;
    const long col = wid % ncol;
    const int i = int(col % g.nx), j = int(col / g.nx);
    const float h = float(g.h);
    const float xf = float((i - 0.5 * (g.nx - 1)) * g.h), yf = float((j - 0.5 * (g.ny - 1)) * g.h);
    const float cuf = 0.5f * float(g.nu - 1), cvf = 0.5f * float(g.nv - 1);
    const float invdu = float(1.0 / g.du);
    const bool cone = g.mode == CTK_CONE3D;
    float zk[KZ], acc[KZ];
#pragma unroll
    for (int m = 0; m < KZ; ++m) {
        const int k = kb + lane + 32 * m;
        zk[m] = float((k - 0.5 * (g.nz - 1)) * g.h);
        acc[m] = 0.f;
    }
    for (int a = 0; a < g.na; ++a) {
        const double2 tr = g.ctst[a];
        const float ct = float(tr.x), st = float(tr.y);
        float fu, t = 1.f, rx = 0.f, ry = 0.f, scale_par = 0.f;
        if (cone) {
            const float sx = float(g.dso) * ct, sy = float(g.dso) * st;
            rx = xf - sx;
            ry = yf - sy;
            const float depth = -(rx * ct + ry * st);
            if (depth <= 0.f) continue;
            t = float(g.dso + g.dod) / depth;
            const float px = sx + t * rx, py = sy + t * ry;
            fu = (-px * st + py * ct) * invdu + cuf;
        } else {
            fu = (-xf * st + yf * ct) * invdu + cuf;
            scale_par = h / fmaxf(fabsf(ct), fabsf(st));
        }
        const float fiu = floorf(fu);
        const int iu = int(fiu);
        const float tu = fu - fiu;
        if (iu < -1 || iu >= g.nu) continue;
        const bool u0ok = iu >= 0, u1ok = iu + 1 < g.nu;
        const float* c0 = pt + size_t(a * g.nu + iu) * g.nv;
        const float* c1 = c0 + g.nv;
        const float arxy = fmaxf(fabsf(rx), fabsf(ry));
        const float rxy2 = rx * rx + ry * ry;
#pragma unroll
        for (int m = 0; m < KZ; ++m) {
            const int k = kb + lane + 32 * m;
            if (k >= g.nz) break;
            const float z = zk[m];
            const float fv = (g.nv == 1) ? 0.f : fmaf(t * z, invdu, cvf);
            const float fiv = floorf(fv);
            const int iv = int(fiv);
            const float tv = fv - fiv;
            const bool v0ok = iv >= 0 && iv < g.nv, v1ok = iv + 1 >= 0 && iv + 1 < g.nv;
            const float p00 = (u0ok && v0ok) ? __ldg(c0 + iv) : 0.f;
            const float p10 = (u1ok && v0ok) ? __ldg(c1 + iv) : 0.f;
            const float p01 = (u0ok && v1ok) ? __ldg(c0 + iv + 1) : 0.f;
            const float p11 = (u1ok && v1ok) ? __ldg(c1 + iv + 1) : 0.f;
            const float s0 = fmaf(tu, p10 - p00, p00);
            const float s1 = fmaf(tu, p11 - p01, p01);
            const float sample = fmaf(tv, s1 - s0, s0);
            float scale;
            if (cone) {
                const float dom = fmaxf(arxy, fabsf(z));
                scale = h * sqrtf(rxy2 + z * z) / dom;
            } else {
                scale = scale_par;
            }
            acc[m] = fmaf(scale, sample, acc[m]);
        }
    }
#pragma unroll
    for (int m = 0; m < KZ; ++m) {
        const int k = kb + lane + 32 * m;
        if (k < g.nz) x[size_t(i) + size_t(g.nx) * (size_t(j) + size_t(g.ny) * k)] = acc[m];
    }
}

int pick_kz(int nz) {
    if (nz <= 32) return 1;
    if (nz <= 64) return 2;
    if (nz <= 128) return 4;
    if (nz <= 256) return 8;
    return 16;
}

void build_quads(Geometry& g, const float* x, cudaStream_t s) {
    const size_t nqx = size_t(g.nx) * (size_t(g.ny) + 1) * (size_t(g.nz) + 1);
    const size_t nqy = size_t(g.ny) * (size_t(g.nx) + 1) * (size_t(g.nz) + 1);
    g.vx.ensure(nqx * sizeof(float4));
    g.vy.ensure(nqy * sizeof(float4));
    {
        dim3 blk(32, 8), grd((g.nx + 31) / 32, (g.ny + 1 + 31) / 32, g.nz + 1);
        k_quads_x<<<grd, blk, 0, s>>>(g.nx, g.ny, g.nz, x, g.vx.as<float4>());
        after_launch("k_quads_x");
    }
    {
        dim3 blk(128), grd((g.nx + 1 + 127) / 128, g.nz + 1, g.ny);
        k_quads_y<<<grd, blk, 0, s>>>(g.nx, g.ny, g.nz, x, g.vy.as<float4>());
        after_launch("k_quads_y");
    }
}

template <bool SCALE>
void transpose_proj(Geometry& g, const float* y, cudaStream_t s) {
    g.proj_t.ensure(g.range() * sizeof(float));
    dim3 blk(32, 8), grd((g.nu + 31) / 32, (g.nv + 31) / 32, g.na);
    k_proj_transpose<SCALE><<<grd, blk, 0, s>>>(g.kgeom(), y, g.proj_t.as<float>());
    after_launch("k_proj_transpose");
}

template <int CLASS>
void launch_plane(Geometry& g, float* x, cudaStream_t s) {
    const int nh = CLASS ? g.nx : g.ny;
    const int planes = CLASS ? g.ny : g.nx;
    const int ptiles = (nh + BP_PB - 1) / BP_PB;
    const int kbands = (g.nz + BP_KB - 1) / BP_KB;
    const size_t smem = sizeof(float) * (size_t(BP_PB) * BP_KB + size_t(BP_PB) * BP_SL + 2 * BP_PB + g.nv);
    static size_t configured = 0;
    if (smem > configured) {
        CTK_CUDA(cudaFuncSetAttribute(k_atb_plane_f32<CLASS>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        configured = smem;
    }
    dim3 grd(unsigned(ptiles * kbands), unsigned(planes));
    k_atb_plane_f32<CLASS><<<grd, BP_PB, smem, s>>>(g.kgeom(), g.proj_t.as<float>(), x, ptiles);
    after_launch("k_atb_plane_f32");
}

template <int KZ>
void launch_voxel(Geometry& g, float* x, cudaStream_t s) {
    const int kblocks = (g.nz + 32 * KZ - 1) / (32 * KZ);
    const long warps = long(g.nx) * g.ny * kblocks;
    dim3 blk(32, 4);
    const unsigned grd = unsigned((warps + 3) / 4);
    k_atb_voxel_f32<KZ><<<grd, blk, 0, s>>>(g.kgeom(), g.proj_t.as<float>(), x, kblocks);
    after_launch("k_atb_voxel_f32");
}

dim3 fwd_grid(const Geometry& g) { return dim3((g.nu + FWD_BX - 1) / FWD_BX, (g.nv + FWD_BY - 1) / FWD_BY, g.na); }

}  // namespace

void ax_f32(Geometry& g, const float* x, float* y, cudaStream_t s) {
    build_quads(g, x, s);
    CTK_CUDA(cudaEventRecord(g.ev0, s));
    k_ax_f32<false><<<fwd_grid(g), dim3(FWD_BX, FWD_BY), 0, s>>>(g.kgeom(), g.vx.as<float4>(), g.vy.as<float4>(), x, y,
                                                                 nullptr, nullptr);
    after_launch("k_ax_f32");
    CTK_CUDA(cudaEventRecord(g.ev1, s));
}

void ax_residual_f32(Geometry& g, const float* x, const float* b, double* d_out, cudaStream_t s) {
    build_quads(g, x, s);
    const dim3 grd = fwd_grid(g);
    const size_t nblk = size_t(grd.x) * grd.y * grd.z;
    g.proj_t.ensure(std::max(g.range() * sizeof(float), nblk * sizeof(double)));
    double* partials = g.proj_t.as<double>();
    CTK_CUDA(cudaEventRecord(g.ev0, s));
    k_ax_f32<true><<<grd, dim3(FWD_BX, FWD_BY), 0, s>>>(g.kgeom(), g.vx.as<float4>(), g.vy.as<float4>(), x, nullptr, b,
                                                        partials);
    after_launch("k_ax_f32_residual");
    CTK_CUDA(cudaEventRecord(g.ev1, s));
    finish_sum(partials, int(nblk), d_out, s);
}

void atb_matched_f32(Geometry& g, const float* y, float* x, cudaStream_t s) {
    transpose_proj<true>(g, y, s);
    CTK_CUDA(cudaEventRecord(g.ev0, s));
    launch_plane<0>(g, x, s);
    launch_plane<1>(g, x, s);
    CTK_CUDA(cudaEventRecord(g.ev1, s));
    if (g.has_zrays) {
        const size_t n = g.domain();
        k_atb_matched_zrays_f32<<<unsigned((n + 127) / 128), 128, 0, s>>>(g.kgeom(), g.proj_t.as<float>(), x);
        after_launch("k_atb_matched_zrays_f32");
    }
}

void atb_voxel_f32(Geometry& g, const float* y, float* x, cudaStream_t s) {
    transpose_proj<false>(g, y, s);
    CTK_CUDA(cudaEventRecord(g.ev0, s));
    switch (pick_kz(g.nz)) {
        case 1: launch_voxel<1>(g, x, s); break;
        case 2: launch_voxel<2>(g, x, s); break;
        case 4: launch_voxel<4>(g, x, s); break;
        case 8: launch_voxel<8>(g, x, s); break;
        default: launch_voxel<16>(g, x, s); break;
    }
    CTK_CUDA(cudaEventRecord(g.ev1, s));
}

}  // namespace ctkb
