// Joseph forward projection Ax for T = float (projector.hpp:113-162) on sm_100a.
//
// Layouts in HBM (f32, z fastest, zero-padded so the four bilinear taps need no checks):
//   wx[i][j+2][k+2]  one plane per x-slice, h = y   (x-dominant rays walk x)
//   wy[j][i+2][k+2]  one plane per y-slice, h = x   (y-dominant rays walk y)
// All rays of one detector column share fh(s) exactly (it depends on the column only), so
// a warp = 32 consecutive detector ROWS of one column has one in-plane index ih per slice
// and consecutive z indices: each tap load of the warp is one contiguous z run (1-2 lines).
//
// L2 reuse.  The volume (512 MiB at 512^3) does not fit the 126 MB L2 and every view
// crosses all of it.  Each ray's slices are split into chunks, one launch per chunk (in
// order, accumulating into y); inside a launch blocks are dispatched with the detector-row
// band SLOWEST and views class by class (x-dominant first), so the resident blocks cover
// every view of one (band, chunk), whose samples stay in one ~26 MB slab of one layout copy:
// that slab comes from HBM about once per launch instead of once per view.
//
// Samples are taken two slices at a time in packed f32x2 arithmetic (FFMA2 / FADD2.RM).
#include <climits>
#include <cstdlib>

#include "f32_common.cuh"

namespace ctkb {
namespace {

// ---- z-fastest variant ------------------------------------------------------------------
// All rays of one detector column share fh(s) exactly (it depends on the column only), so a
// warp of 32 consecutive detector ROWS of one column has a single in-plane index ih per
// slice and consecutive z indices.  With the layouts stored z-fastest,
//   wx[i][j+2][k+2]  (x-dominant rays: slice i, h = j)     wy[j][i+2][k+2]  (h = i)
// each of the 4 tap loads of a warp covers one contiguous z run (1-2 cache lines) instead
// of two partial rows of a y/x-fastest plane.
// Block = 32 detector rows x CTK_FWD_BC columns.  4 columns (128 threads) capped at 56
// registers (9 blocks = 36 warps per SM; a few bytes of spill outside the slice loop):
// 48.4 vs 49.9 ms at C3 with 8 columns / 64 registers / 32 warps, 3.35 vs 3.45 ms at
// 256^3/180, 273 vs 278 ms at 1024^3/200 -- the loop is latency-bound, occupancy pays
#ifndef CTK_FWD_BC
#define CTK_FWD_BC 4
#endif
#ifndef CTK_FWD_CHUNKS
#define CTK_FWD_CHUNKS 2  // minimum slice chunks per ray (fwd_chunks); 64.8 -> 50.4 ms at 512^3 vs unchunked
#endif
#ifndef CTK_FWD_UNROLL
#define CTK_FWD_UNROLL 1
#endif
#ifndef CTK_FWD_MINB
#define CTK_FWD_MINB 9  // minimum resident blocks per SM for the register allocator (56 registers)
#endif
#ifndef CTK_FWD2_MINB
#define CTK_FWD2_MINB 6  // the two-volume march: 80 registers, 6 CTAs/SM (69.2 ms per pair at C3; 81.2 at 8 CTAs / 64 registers, 74.1 at 9 with spills)
#endif
#ifndef CTK_FWD2_UNROLL
#define CTK_FWD2_UNROLL 1
#endif
constexpr int kFwd2Unroll = CTK_FWD2_UNROLL;
constexpr int ZW_BR = 32, ZW_BC = CTK_FWD_BC, kFwdUnroll = CTK_FWD_UNROLL;  // block: 32 detector rows (lanes) x ZW_BC columns
// zero guard planes on each side of the z-fast layouts (h and z): a tap index may step one
// beyond the contributing range where anchored positions round across a voxel boundary
constexpr int kPad = 2;

__device__ __forceinline__ const float* opaque_ptr(const float* p) {
    asm("" : "+l"(p));
    return p;
}

__device__ __forceinline__ const float2* opaque_ptr2(const float2* p) {
    asm("" : "+l"(p));
    return p;
}

// x[i + nx(j + ny k)] -> wx[i][j+kPad][k+kPad] and wy[j][i+kPad][k+kPad]: 32x32 (i, k) tile
// transposes
__global__ void k_relayout_zfast(int nx, int ny, int nz, const float* __restrict__ x, float* __restrict__ wx,
                                 float* __restrict__ wy) {
    __shared__ float tile[32][33];
    const int i0 = blockIdx.x * 32, k0 = blockIdx.y * 32, j = blockIdx.z;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int i = i0 + threadIdx.x, k = k0 + r;
        tile[r][threadIdx.x] = (i < nx && k < nz) ? __ldg(x + size_t(i) + size_t(nx) * (j + size_t(ny) * k)) : 0.f;
    }
    __syncthreads();
    const size_t pz = size_t(nz) + 2 * kPad;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int i = i0 + r, k = k0 + threadIdx.x;
        if (i < nx && k < nz) {
            const float v = tile[threadIdx.x][r];
            wx[(size_t(i) * (ny + 2 * kPad) + (j + kPad)) * pz + k + kPad] = v;
            wy[(size_t(j) * (nx + 2 * kPad) + (i + kPad)) * pz + k + kPad] = v;
        }
    }
}

// Siddon sum of one ray over its slabs (f32_common.cuh), before the factor L = ray_step:
// sum over slabs of min(cy,cz) v(ja,ka) + (cy-min) v(ja,ka+sz) + (cz-min) v(ja+sy,ka)
// + (1-max) v(ja+sy,ka+sz), with (ja, ka) the cells at the slab's s - 1/2 boundary.
__device__ __forceinline__ float fma_v(float w, float v, float acc) { return fmaf(w, v, acc); }
__device__ __forceinline__ float2 fma_v(float w, float2 v, float2 acc) {  // per volume, the scalar op
    return make_float2(fmaf(w, v.x, acc.x), fmaf(w, v.y, acc.y));
}

// V = float: one volume; V = float2: two interleaved volumes (k_ax2_zfast_f32), each with
// exactly the one-volume operation sequence
template <class Off, class V>
__device__ V siddon_ray(const KGeom& g, const double4& c64, float fhd, int nh, int ns, const V* base, Off pz,
                        Off plane, float vd, float czf, float vr, int nch, int chunk) {
    const float Wd = z_cross(g, c64), fcs = sid_fc(g);
    const int izs = sid_izc(g);
    const float dz = vr * Wd;
    const bool incy = fhd >= 0.f, incz = dz >= 0.f;
    // 1/|fhd| and 1/|vr Wd| = (1/|vr|)(1/|Wd|), as the transpose forms them
    const float ay = __frcp_rn(fabsf(fhd)), az = __frcp_rn(fabsf(vr)) * __frcp_rn(fabsf(Wd));
    const Off dy = incy ? pz : -pz, dz1 = incz ? 1 : -1;
    const float2 aby = sid_coef(incy, ay), abz = sid_coef(incz, az);
    using U = typename std::conditional<sizeof(Off) == 4, unsigned, unsigned long long>::type;
    const U upz = U(pz), uplane = U(plane);
    // cells (j, k) at the slab's t = 0 boundary, the expressions of the transpose
    auto cell0 = [&](int s, int& j, int& k) {
        const int sc = slice_centre(s);
        int jA, jr;
        float tA, Whi, Wr, fy;
        double G;
        sid_anchor(c64, sc, jA, tA, G);
        z_split(g, G, Whi, Wr);
        const float kb = float(s - sc) - 0.5f;
        split(fmaf(kb, fhd, tA), jr, fy);
        const float tt = split_t(fmaf(vr, fmaf(kb, Wd, Wr), fmaf(vr, Whi, fcs)));
        j = jA + jr;
        k = izs + (__float_as_int(tt) - kSplitBias) - g.z0;
    };
    // a slab contributes iff a cell is inside: j in [-1, nh] and k in [-1, nz] (the other
    // cell is then within the two guard planes); find the interval like the Joseph march
    auto inside = [&](int s) {
        int j, k;
        cell0(s, j, k);
        return j >= -1 && j <= nh && k >= -1 && k <= g.nz;
    };
    int s0 = 0, s1 = ns - 1;
    clip_affine(c64.x + 0.5 - 0.5 * c64.y, c64.y, -1.0, nh + 1.0, s0, s1);
    clip_affine(double(vd) * (c64.z - 0.5 * c64.w) + czf + 0.5 - g.z0, double(vd) * c64.w, -1.0, g.nz + 1.0, s0, s1);
    while (s0 <= s1 && !inside(s0)) ++s0;
    while (s1 >= s0 && !inside(s1)) --s1;
    if (s0 <= s1) {
        while (s0 > 0 && inside(s0 - 1)) --s0;
        while (s1 < ns - 1 && inside(s1 + 1)) ++s1;
    }
    if (nch > 1) {
        const int len = (ns + nch - 1) / nch;
        s0 = max(s0, chunk * len);
        s1 = min(s1, chunk * len + len - 1);
    }
#ifdef CTK_CHECKED
    const long long lay_n = (long long)ns * (long long)plane, base_abs = (long long)(kPad * pz + kPad);
#endif
    V acc;
    if constexpr (sizeof(V) == 4) acc = 0.f;
    else acc = make_float2(0.f, 0.f);
    for (int s = s0; s <= s1;) {  // slice blocks: fp64 anchors once per block
        const int sc = slice_centre(s);
        const int se = min(s1, sc + kSB / 2 - 1);
        int jA;
        float tA, Whi, Wr;
        double G;
        sid_anchor(c64, sc, jA, tA, G);
        z_split(g, G, Whi, Wr);
        const float S = fmaf(vr, Whi, fcs);  // exact
        // offsets from the raw bits of the split sums (j + bias, k + bias), in modular arithmetic
        const U rb = U(Off(jA)) * upz + U(Off(izs - g.z0)) - U(kSplitBias) * (upz + 1u);
        // one slab: its t = 0 boundary at kb (relative to sc) split into cells and fractions
        // (ty, fy: in-plane; tt, fz: z), then the four cells' chord weights
        auto slab = [&](int sl, float ty, float fy, float tt, float fz) {
            const float cy = sid_cross(fy, aby), cz = sid_cross(fz, abz);
            const float m = fminf(cy, cz), M = fmaxf(cy, cz);
            Off o = Off(U(sl) * uplane + rb + U(unsigned(__float_as_int(ty))) * upz + U(unsigned(__float_as_int(tt))));
#ifdef CTK_CHECKED
            if (base_abs + (long long)o - (long long)pz - 1 < 0 || base_abs + (long long)o + (long long)pz + 1 >= lay_n) {
                atomicOr(g.chk, 1u << 0);
                o = Off(pz + 1 - base_abs);
            }
#endif
            // the second cells are one step in the ray's directions, offset only when the
            // boundary is crossed (their weights are exactly 0 otherwise; measured at 256^3/180:
            // 5.22 ms, against 5.62 loading the four distinct cells always and 6.05 predicating
            // the second-cell loads)
            const bool xy = cy < 1.f, xz = cz < 1.f;
            const Off o01 = o + (xz ? dz1 : Off(0)), o10 = o + (xy ? dy : Off(0)), o11 = o10 + (xz ? dz1 : Off(0));
            const V v00 = __ldg(base + o), v01 = __ldg(base + o01), v10 = __ldg(base + o10), v11 = __ldg(base + o11);
            acc = fma_v(m, v00, acc);        // (ja, ka)
            acc = fma_v(cy - m, v01, acc);   // (ja, kb)
            acc = fma_v(cz - m, v10, acc);   // (jb, ka)
            acc = fma_v(1.f - M, v11, acc);  // (jb, kb)
        };
        // two slabs at a time: boundary positions in packed f32x2 arithmetic (per lane the
        // scalar sequence of the transpose: fmaf, split_t, exact fraction)
        float2 kb2 = make_float2(float(s - sc) - 0.5f, float(s - sc) + 0.5f);
        const float2 fhd2 = make_float2(fhd, fhd), tA2 = make_float2(tA, tA), Wd2 = make_float2(Wd, Wd);
        const float2 Wr2 = make_float2(Wr, Wr), vr2 = make_float2(vr, vr), S2 = make_float2(S, S);
        const float2 M2 = make_float2(kSplitM, kSplitM), nM2 = make_float2(-kSplitM, -kSplitM);
        const float2 m1 = make_float2(-1.f, -1.f), two = make_float2(2.f, 2.f);
        for (; s + 1 <= se; s += 2) {
            const float2 fyr = __ffma2_rn(kb2, fhd2, tA2);
            const float2 ty = __fadd2_rd(fyr, M2);
            const float2 fy = __ffma2_rn(__fadd2_rn(ty, nM2), m1, fyr);
            const float2 wlo = __ffma2_rn(kb2, Wd2, Wr2);
            const float2 tt = __fadd2_rd(__ffma2_rn(vr2, wlo, S2), M2);
            const float2 fz = __ffma2_rn(vr2, wlo, __ffma2_rn(__fadd2_rn(tt, nM2), m1, S2));
            kb2 = __fadd2_rn(kb2, two);
            slab(s, ty.x, fy.x, tt.x, fz.x);
            slab(s + 1, ty.y, fy.y, tt.y, fz.y);
        }
        if (s <= se) {  // odd count: the block's last slab, scalar
            const float kb = kb2.x;
            const float fyr = fmaf(kb, fhd, tA);
            const float ty = split_t(fyr);
            const float wlo = fmaf(kb, Wd, Wr);
            const float tt = split_t(fmaf(vr, wlo, S));
            slab(s, ty, split_frac(fyr, ty), tt, fmaf(vr, wlo, fmaf(__fsub_rn(tt, kSplitM), -1.f, S)));
            ++s;
        }
    }
    return acc;
}

// MODE 0: y = A x.   MODE 1: per-block partial of sum (A x - b)^2 (y never stored).
// nch > 1 (MODE 0 only): slice chunking for L2 locality -- one launch per chunk of the
// slices, in chunk order; chunk 0 writes y and later chunks add their partial sums to it
// (deterministic: the launches are ordered on the stream).
// SID = 1: the f32 Siddon model (f32_common.cuh) on the same layouts: per slab the four
// cells (ja|ja+sy, ka|ka+sz) of the chord instead of the four bilinear taps.
template <int MODE, class Off, int SID = 0, int WIN = 0>
__global__ void __launch_bounds__(ZW_BR * ZW_BC, CTK_FWD_MINB)
k_ax_zfast_f32(KGeom g, const int* __restrict__ vorder, const float* __restrict__ wx, const float* __restrict__ wy,
               const float* __restrict__ xs, float* __restrict__ y, const float* __restrict__ b,
               double* __restrict__ partials, int nch, int chunk, int band0) {
    // WIN: the band-sharded range's row window; else the whole detector (constants)
    const int W0 = WIN ? g.w0 : 0, NW = WIN ? g.nw : g.nv;
    __shared__ float outs[ZW_BR][ZW_BC + 1];
    const int band = blockIdx.z + band0;
    const int iv = band * ZW_BR + threadIdx.x;
    const int a = vorder[blockIdx.y];
    const int iu = blockIdx.x * ZW_BC + threadIdx.y;
    float out = 0.f;
    const bool live = iu < g.nu && iv < g.nv && iv >= W0 && iv < W0 + NW;  // rows held (band-sharded range)
    if (live) {
        const int c = a * g.nu + iu;
        const double2 cs = g.colstep[c];
        const double v = row_coord(g, iv);
        if (g.has_zrays && is_zray(g, cs, v)) {
            if (SID) {
                // Siddon z-rays: the exact DDA (siddon.cu, zonly) fills them after this launch
            } else if (chunk == 0) {  // z-rays are marched whole by the first chunk
                const double2 tr = g.ctst[a];
                WalkF w;
                walk_generic(g, tr.x, tr.y, iu, iv, w);
                out = march_generic(g, w, xs);
            }
        } else {
            const float4 cd = g.col[c];
            const double4 c64 = g.col64[c];
            const int A = g.colaxis[c];
            const int nh = A ? g.nx : g.ny;
            const int ns = A ? g.ny : g.nx;
            const Off pz = g.nz + 2 * kPad;
            const Off plane = pz * Off(nh + 2 * kPad);
            // tap (h, z) of slice s at base[s*plane + h*pz + (z - z0)]
            const float* base = (A ? wy : wx) + kPad * pz + kPad;
            const float vd = float(v);
            const float czf = 0.5f * float(g.nzg - 1);  // global z centre; slab slices start at z0
            const unsigned unh = unsigned(nh), unz = unsigned(g.nz);
            if constexpr (SID) {
                out = siddon_ray(g, c64, cd.y, nh, ns, base, pz, plane, vd, czf, row_vr(g, iv), nch, chunk) *
                      ray_step(g, cs, v);
            } else {
            // anchored positions (f32_common.cuh): per slice block the fp64 anchors, per lane
            // the exact row term S
            const float Wd = z_cross(g, c64), vr = row_vr(g, iv), fc = cz_frac(g);
            const int izc = cz_int(g);
            auto pos = [&](int s, int& ih, int& iz) {
                const int sc = slice_centre(s);
                int ihA, a, b;
                float thA, Whi, Wr, t0, t1;
                double G;
                slice_anchor(c64, sc, ihA, thA, G);
                z_split(g, G, Whi, Wr);
                const float kf = float(s - sc);
                split(fmaf(kf, cd.y, thA), a, t0);
                split(fmaf(vr, fmaf(kf, Wd, Wr), fmaf(vr, Whi, fc)), b, t1);
                ih = ihA + a;
                iz = izc + b;
            };
            // a sample contributes iff some tap is inside the volume: ih in [-1, nh-1] and
            // iz in [-1, nz-1].  ih(s) and iz(s) are monotone in s up to the rounding of the
            // anchored offsets, so the contributing slices form one interval; find its ends
            // exactly with the kernel's own arithmetic, starting from the fp64 estimate.  (A
            // slice inside the interval can sit one index beyond the volume when a position
            // lies within rounding of a voxel boundary: the layouts carry two zero guard
            // planes on each side, so its taps read zeros.)
            auto inside = [&](int s) {
                int ih, iz;
                pos(s, ih, iz);
                return unsigned(ih + 1) <= unh && unsigned(iz - g.z0 + 1) <= unz;
            };
            int s0 = 0, s1 = ns - 1;
            clip_affine(cd.x, cd.y, -1.0, nh, s0, s1);
            clip_affine(double(vd) * cd.z + czf - g.z0, double(vd) * cd.w, -1.0, g.nz, s0, s1);
            while (s0 <= s1 && !inside(s0)) ++s0;
            while (s1 >= s0 && !inside(s1)) --s1;
            if (s0 <= s1) {
                while (s0 > 0 && inside(s0 - 1)) --s0;
                while (s1 < ns - 1 && inside(s1 + 1)) ++s1;
            }
            if (nch > 1) {
                const int len = (ns + nch - 1) / nch;
                s0 = max(s0, chunk * len);
                s1 = min(s1, chunk * len + len - 1);
            }
            float acc = 0.f;
            // Offsets are formed from the raw bit patterns of the split sums (ih + bias,
            // iz + bias); the bias and the anchors are folded into the running slice offset,
            // in unsigned (modular) arithmetic, so a sample costs one IMAD and no
            // float->int conversion.
            using U = typename std::conditional<sizeof(Off) == 4, unsigned, unsigned long long>::type;
            const U upz = U(pz), uplane = U(plane), uplane2 = uplane + uplane;
            const U cbias = U(kSplitBias) * (upz + 1u) + U(unsigned(g.z0)) - U(unsigned(izc));
            // tap row ih+1; opaque so each tap row costs one IMAD.WIDE rather than a
            // sign-extended 64-bit add chain on (off + pz)
            const float* base1 = opaque_ptr(base + pz);
            // Two slices per iteration in packed f32x2 arithmetic (FFMA2 / FADD2 on sm_100a):
            // every lane of a pair performs exactly the scalar operation sequence, so the
            // positions, floors and weights are bit-identical to the matched backprojector's;
            // only the ray sum is split into even / odd slices.
            const float2 fhd2 = make_float2(cd.y, cd.y), Wd2 = make_float2(Wd, Wd), vr2 = make_float2(vr, vr);
            const float2 M2 = make_float2(kSplitM, kSplitM), nM2 = make_float2(-kSplitM, -kSplitM);
            const float2 m1 = make_float2(-1.f, -1.f), two = make_float2(2.f, 2.f);
            float2 acc2 = make_float2(0.f, 0.f);
#ifdef CTK_CHECKED
            // checked build: the four taps o, o+1, o+pz, o+pz+1 must lie inside the layout
            const long long lay_n = (long long)ns * (long long)plane, base_abs = (long long)(kPad * pz + kPad);
            auto chk_tap = [&](Off o) -> Off {
                const long long lo = base_abs + (long long)o;
                if (lo < 0 || lo + (long long)pz + 1 >= lay_n) {
                    atomicOr(g.chk, 1u << 0);
                    return Off(-base_abs);
                }
                return o;
            };
#else
            auto chk_tap = [](Off o) { return o; };
#endif
            for (int s = s0; s <= s1;) {  // slice blocks
                const int sc = slice_centre(s);
                const int se = min(s1, sc + kSB / 2 - 1);
                int ihA;
                float thA, Whi, Wr;
                double G;
                slice_anchor(c64, sc, ihA, thA, G);
                z_split(g, G, Whi, Wr);
                const float S = fmaf(vr, Whi, fc);  // exact
                // U(Off(ihA)): sign-extended, ihA < 0 at the volume edge (a 64-bit U must not zero-extend)
                U sb = U(s) * uplane + U(Off(ihA)) * upz - cbias;
                const float2 thA2 = make_float2(thA, thA), Wr2 = make_float2(Wr, Wr), S2 = make_float2(S, S);
                float2 k2 = make_float2(float(s - sc), float(s - sc + 1));
                const int cnt = se - s + 1;
#pragma unroll kFwdUnroll
                for (int np = cnt >> 1; np > 0; --np) {
                    const float2 fh = __ffma2_rn(k2, fhd2, thA2);
                    const float2 wlo = __ffma2_rn(k2, Wd2, Wr2);
                    const float2 tht = __fadd2_rd(fh, M2);
                    const float2 tzt = __fadd2_rd(__ffma2_rn(vr2, wlo, S2), M2);
                    const float2 th = __ffma2_rn(__fadd2_rn(tht, nM2), m1, fh);  // fh - floor(fh)
                    const float2 tz = __ffma2_rn(vr2, wlo, __ffma2_rn(__fadd2_rn(tzt, nM2), m1, S2));
                    const Off o0 =
                        chk_tap(Off(U(unsigned(__float_as_int(tht.x))) * upz + (sb + U(unsigned(__float_as_int(tzt.x))))));
                    const Off o1 = chk_tap(
                        Off(U(unsigned(__float_as_int(tht.y))) * upz + (sb + uplane + U(unsigned(__float_as_int(tzt.y))))));
                    k2 = __fadd2_rn(k2, two);
                    sb += uplane2;
                    const float* p0 = base + o0;
                    const float* q0 = base1 + o0;
                    const float* p1 = base + o1;
                    const float* q1 = base1 + o1;
                    const float2 v00 = make_float2(__ldg(p0), __ldg(p1)), v01 = make_float2(__ldg(p0 + 1), __ldg(p1 + 1));
                    const float2 v10 = make_float2(__ldg(q0), __ldg(q1)), v11 = make_float2(__ldg(q0 + 1), __ldg(q1 + 1));
                    const float2 a0 = __ffma2_rn(th, __ffma2_rn(v00, m1, v10), v00);
                    const float2 a1 = __ffma2_rn(th, __ffma2_rn(v01, m1, v11), v01);
                    acc2 = __fadd2_rn(acc2, __ffma2_rn(tz, __ffma2_rn(a0, m1, a1), a0));
                }
                if (cnt & 1) {  // odd count: the block's last slice, scalar
                    const float kf = k2.x;
                    const float fh = fmaf(kf, cd.y, thA);
                    const float wlo = fmaf(kf, Wd, Wr);
                    const float tht = split_t(fh), tzt = split_t(fmaf(vr, wlo, S));
                    const float th = split_frac(fh, tht);
                    const float tz = fmaf(vr, wlo, fmaf(__fsub_rn(tzt, kSplitM), -1.f, S));
                    const Off off =
                        chk_tap(Off(U(unsigned(__float_as_int(tht))) * upz + (sb + U(unsigned(__float_as_int(tzt))))));
                    const float* p = base + off;
                    const float* q = base1 + off;
                    const float v00 = __ldg(p), v01 = __ldg(p + 1);  // (ih, iz), (ih, iz+1)
                    const float v10 = __ldg(q), v11 = __ldg(q + 1);  // (ih+1, iz), (ih+1, iz+1)
                    const float a0 = fmaf(th, v10 - v00, v00);
                    const float a1 = fmaf(th, v11 - v01, v01);
                    acc += fmaf(tz, a1 - a0, a0);
                }
                s = se + 1;
            }
            acc += acc2.x + acc2.y;
            const float stp = ray_step(g, cs, v);
            out = stp * acc;
            }
        }
    }
    if (MODE == 0) {
        // transpose through shared memory so the stores run along detector columns
        outs[threadIdx.x][threadIdx.y] = out;
        __syncthreads();
        const int t = threadIdx.x + ZW_BR * threadIdx.y;
        const int r = t / ZW_BC, cc = t % ZW_BC;
        const int ivw = band * ZW_BR + r, iuw = blockIdx.x * ZW_BC + cc;
        if (ivw >= W0 && ivw < W0 + NW && iuw < g.nu) {
            float* yo = y + (size_t(a) * NW + size_t(ivw - W0)) * g.nu + iuw;
            *yo = chunk == 0 ? outs[r][cc] : *yo + outs[r][cc];
        }
    }
    if (MODE != 0) {
        double rr = 0.0;
        if (live) {
            const double d = double(out) - double(__ldg(b + (size_t(a) * NW + size_t(iv - W0)) * g.nu + iu));
            rr = d * d;
        }
        rr = block_sum(rr);
        if (threadIdx.x == 0 && threadIdx.y == 0)
            partials[(size_t(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = rr;
    }
}

// Two volumes through one ray march (y1 = A x1, y2 = A x2; f32 Joseph, whole volume).  The
// solvers need A v for the next Krylov step and A x for the explicit residual of the
// iteration just finished (solve_log.hpp:102-115); both exist at the same time, and their
// samples share every position, floor and weight.  The layouts hold the two volumes
// interleaved (float2: .x from x1, .y from x2), so one 8-byte tap load serves both, and
// per volume the operation sequence is exactly k_ax_zfast_f32's (slice pairs: even slices
// in one accumulator, odd in the other, the odd tail scalar), so each output is
// bit-identical to a single-volume launch with the same chunking.
template <class Off, int SID>
__global__ void __launch_bounds__(ZW_BR * ZW_BC, CTK_FWD2_MINB)
k_ax2_zfast_f32(KGeom g, const int* __restrict__ vorder, const float2* __restrict__ wx, const float2* __restrict__ wy,
                const float* __restrict__ xs1, const float* __restrict__ xs2, float* __restrict__ y1,
                float* __restrict__ y2, int nch, int chunk) {
    __shared__ float outs[2][ZW_BR][ZW_BC + 1];
    const int band = blockIdx.z;
    const int iv = band * ZW_BR + threadIdx.x;
    const int a = vorder[blockIdx.y];
    const int iu = blockIdx.x * ZW_BC + threadIdx.y;
    float out1 = 0.f, out2 = 0.f;
    if (iu < g.nu && iv < g.nv) {
        const int c = a * g.nu + iu;
        const double2 cs = g.colstep[c];
        const double v = row_coord(g, iv);
        if (g.has_zrays && is_zray(g, cs, v)) {
            if (SID) {
                // Siddon z-rays: the exact DDA fills them after the launches (as ax_f32)
            } else if (chunk == 0) {
                const double2 tr = g.ctst[a];
                WalkF w;
                walk_generic(g, tr.x, tr.y, iu, iv, w);
                out1 = march_generic(g, w, xs1);
                out2 = march_generic(g, w, xs2);
            }
        } else {
            const float4 cd = g.col[c];
            const double4 c64 = g.col64[c];
            const int A = g.colaxis[c];
            const int nh = A ? g.nx : g.ny;
            const int ns = A ? g.ny : g.nx;
            const Off pz = g.nz + 2 * kPad;
            const Off plane = pz * Off(nh + 2 * kPad);
            const float2* base = (A ? wy : wx) + kPad * pz + kPad;
            const float vd = float(v);
            const float czf = 0.5f * float(g.nzg - 1);
            const unsigned unh = unsigned(nh), unz = unsigned(g.nz);
            if constexpr (SID) {
                const float2 r = siddon_ray(g, c64, cd.y, nh, ns, base, pz, plane, vd, czf, row_vr(g, iv), nch, chunk);
                const float stp = ray_step(g, cs, v);
                out1 = r.x * stp;
                out2 = r.y * stp;
            } else {
            const float Wd = z_cross(g, c64), vr = row_vr(g, iv), fc = cz_frac(g);
            const int izc = cz_int(g);
            // the slice interval of k_ax_zfast_f32 (same arithmetic)
            auto pos = [&](int s, int& ih, int& iz) {
                const int sc = slice_centre(s);
                int ihA, pa, pb;
                float thA, Whi, Wr, t0, t1;
                double G;
                slice_anchor(c64, sc, ihA, thA, G);
                z_split(g, G, Whi, Wr);
                const float kf = float(s - sc);
                split(fmaf(kf, cd.y, thA), pa, t0);
                split(fmaf(vr, fmaf(kf, Wd, Wr), fmaf(vr, Whi, fc)), pb, t1);
                ih = ihA + pa;
                iz = izc + pb;
            };
            auto inside = [&](int s) {
                int ih, iz;
                pos(s, ih, iz);
                return unsigned(ih + 1) <= unh && unsigned(iz + 1) <= unz;
            };
            int s0 = 0, s1 = ns - 1;
            clip_affine(cd.x, cd.y, -1.0, nh, s0, s1);
            clip_affine(double(vd) * cd.z + czf, double(vd) * cd.w, -1.0, g.nz, s0, s1);
            while (s0 <= s1 && !inside(s0)) ++s0;
            while (s1 >= s0 && !inside(s1)) --s1;
            if (s0 <= s1) {
                while (s0 > 0 && inside(s0 - 1)) --s0;
                while (s1 < ns - 1 && inside(s1 + 1)) ++s1;
            }
            if (nch > 1) {
                const int len = (ns + nch - 1) / nch;
                s0 = max(s0, chunk * len);
                s1 = min(s1, chunk * len + len - 1);
            }
            float acc1 = 0.f, acc2 = 0.f;
            using U = typename std::conditional<sizeof(Off) == 4, unsigned, unsigned long long>::type;
            const U upz = U(pz), uplane = U(plane), uplane2 = uplane + uplane;
            const U cbias = U(kSplitBias) * (upz + 1u) - U(unsigned(izc));
            const float2* base1 = opaque_ptr2(base + pz);  // one IMAD.WIDE per tap row
#ifdef CTK_CHECKED
            // checked build: the four taps o, o+1, o+pz, o+pz+1 must lie inside the layout
            const long long lay_n = (long long)ns * (long long)plane, base_abs = (long long)(kPad * pz + kPad);
            auto chk_tap = [&](Off o) -> Off {
                const long long lo = base_abs + (long long)o;
                if (lo < 0 || lo + (long long)pz + 1 >= lay_n) {
                    atomicOr(g.chk, 1u << 0);
                    return Off(-base_abs);
                }
                return o;
            };
#else
            auto chk_tap = [](Off o) { return o; };
#endif
            const float2 fhd2 = make_float2(cd.y, cd.y), Wd2 = make_float2(Wd, Wd), vr2 = make_float2(vr, vr);
            const float2 M2 = make_float2(kSplitM, kSplitM), nM2 = make_float2(-kSplitM, -kSplitM);
            const float2 m1 = make_float2(-1.f, -1.f), two = make_float2(2.f, 2.f);
            // (volume 1, volume 2) of the even and of the odd slices
            float2 accE = make_float2(0.f, 0.f), accO = make_float2(0.f, 0.f);
            for (int s = s0; s <= s1;) {
                const int sc = slice_centre(s);
                const int se = min(s1, sc + kSB / 2 - 1);
                int ihA;
                float thA, Whi, Wr;
                double G;
                slice_anchor(c64, sc, ihA, thA, G);
                z_split(g, G, Whi, Wr);
                const float S = fmaf(vr, Whi, fc);
                U sb = U(s) * uplane + U(Off(ihA)) * upz - cbias;
                const float2 thA2 = make_float2(thA, thA), Wr2 = make_float2(Wr, Wr), S2 = make_float2(S, S);
                float2 k2 = make_float2(float(s - sc), float(s - sc + 1));
                const int cnt = se - s + 1;
#pragma unroll kFwd2Unroll
                for (int np = cnt >> 1; np > 0; --np) {
                    const float2 fh = __ffma2_rn(k2, fhd2, thA2);
                    const float2 wlo = __ffma2_rn(k2, Wd2, Wr2);
                    const float2 tht = __fadd2_rd(fh, M2);
                    const float2 tzt = __fadd2_rd(__ffma2_rn(vr2, wlo, S2), M2);
                    const float2 th = __ffma2_rn(__fadd2_rn(tht, nM2), m1, fh);
                    const float2 tz = __ffma2_rn(vr2, wlo, __ffma2_rn(__fadd2_rn(tzt, nM2), m1, S2));
                    const Off o0 =
                        chk_tap(Off(U(unsigned(__float_as_int(tht.x))) * upz + (sb + U(unsigned(__float_as_int(tzt.x))))));
                    const Off o1 = chk_tap(
                        Off(U(unsigned(__float_as_int(tht.y))) * upz + (sb + uplane + U(unsigned(__float_as_int(tzt.y))))));
                    k2 = __fadd2_rn(k2, two);
                    sb += uplane2;
                    const float2 A00 = __ldg(base + o0), A01 = __ldg(base + o0 + 1);
                    const float2 A10 = __ldg(base1 + o0), A11 = __ldg(base1 + o0 + 1);
                    const float2 B00 = __ldg(base + o1), B01 = __ldg(base + o1 + 1);
                    const float2 B10 = __ldg(base1 + o1), B11 = __ldg(base1 + o1 + 1);
                    {  // even slice: weights th.x, tz.x on both volumes
                        const float2 t = make_float2(th.x, th.x), u = make_float2(tz.x, tz.x);
                        const float2 a0 = __ffma2_rn(t, __ffma2_rn(A00, m1, A10), A00);
                        const float2 a1 = __ffma2_rn(t, __ffma2_rn(A01, m1, A11), A01);
                        accE = __fadd2_rn(accE, __ffma2_rn(u, __ffma2_rn(a0, m1, a1), a0));
                    }
                    {  // odd slice
                        const float2 t = make_float2(th.y, th.y), u = make_float2(tz.y, tz.y);
                        const float2 a0 = __ffma2_rn(t, __ffma2_rn(B00, m1, B10), B00);
                        const float2 a1 = __ffma2_rn(t, __ffma2_rn(B01, m1, B11), B01);
                        accO = __fadd2_rn(accO, __ffma2_rn(u, __ffma2_rn(a0, m1, a1), a0));
                    }
                }
                if (cnt & 1) {
                    const float kf = k2.x;
                    const float fh = fmaf(kf, cd.y, thA);
                    const float wlo = fmaf(kf, Wd, Wr);
                    const float tht = split_t(fh), tzt = split_t(fmaf(vr, wlo, S));
                    const float th = split_frac(fh, tht);
                    const float tz = fmaf(vr, wlo, fmaf(__fsub_rn(tzt, kSplitM), -1.f, S));
                    const Off off =
                        chk_tap(Off(U(unsigned(__float_as_int(tht))) * upz + (sb + U(unsigned(__float_as_int(tzt))))));
                    const float2 v00 = __ldg(base + off), v01 = __ldg(base + off + 1);
                    const float2 v10 = __ldg(base1 + off), v11 = __ldg(base1 + off + 1);
                    {
                        const float a0 = fmaf(th, v10.x - v00.x, v00.x), a1 = fmaf(th, v11.x - v01.x, v01.x);
                        acc1 += fmaf(tz, a1 - a0, a0);
                    }
                    {
                        const float a0 = fmaf(th, v10.y - v00.y, v00.y), a1 = fmaf(th, v11.y - v01.y, v01.y);
                        acc2 += fmaf(tz, a1 - a0, a0);
                    }
                }
                s = se + 1;
            }
            acc1 += accE.x + accO.x;
            acc2 += accE.y + accO.y;
            const float stp = ray_step(g, cs, v);
            out1 = stp * acc1;
            out2 = stp * acc2;
            }
        }
    }
    outs[0][threadIdx.x][threadIdx.y] = out1;
    outs[1][threadIdx.x][threadIdx.y] = out2;
    __syncthreads();
    const int t = threadIdx.x + ZW_BR * threadIdx.y;
    const int r = t / ZW_BC, cc = t % ZW_BC;
    const int ivw = band * ZW_BR + r, iuw = blockIdx.x * ZW_BC + cc;
    if (ivw < g.nv && iuw < g.nu) {
        const size_t o = (size_t(a) * g.nv + size_t(ivw)) * g.nu + iuw;
        y1[o] = chunk == 0 ? outs[0][r][cc] : y1[o] + outs[0][r][cc];
        y2[o] = chunk == 0 ? outs[1][r][cc] : y2[o] + outs[1][r][cc];
    }
}

// x1, x2 -> interleaved wx[i][j+kPad][k+kPad], wy[j][i+kPad][k+kPad] (float2 {x1, x2})
__global__ void k_relayout2_zfast(int nx, int ny, int nz, const float* __restrict__ x1, const float* __restrict__ x2,
                                  float2* __restrict__ wx, float2* __restrict__ wy) {
    __shared__ float2 tile[32][33];
    const int i0 = blockIdx.x * 32, k0 = blockIdx.y * 32, j = blockIdx.z;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int i = i0 + threadIdx.x, k = k0 + r;
        const bool in = i < nx && k < nz;
        const size_t src = size_t(i) + size_t(nx) * (j + size_t(ny) * k);
        tile[r][threadIdx.x] = make_float2(in ? __ldg(x1 + src) : 0.f, in ? __ldg(x2 + src) : 0.f);
    }
    __syncthreads();
    const size_t pz = size_t(nz) + 2 * kPad;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int i = i0 + r, k = k0 + threadIdx.x;
        if (i < nx && k < nz) {
            const float2 v = tile[threadIdx.x][r];
            wx[(size_t(i) * (ny + 2 * kPad) + (j + kPad)) * pz + k + kPad] = v;
            wy[(size_t(j) * (nx + 2 * kPad) + (i + kPad)) * pz + k + kPad] = v;
        }
    }
}

void relayout_zfast(Geometry& g, const float* x, DevBuf& wx, DevBuf& wy, cudaStream_t s) {
    const size_t nwx = size_t(g.nx) * (size_t(g.ny) + 2 * kPad) * (size_t(g.nz_local()) + 2 * kPad);
    const size_t nwy = size_t(g.ny) * (size_t(g.nx) + 2 * kPad) * (size_t(g.nz_local()) + 2 * kPad);
    if (wx.ensure(nwx * sizeof(float))) CTK_CUDA(cudaMemsetAsync(wx.p, 0, nwx * sizeof(float), s));
    if (wy.ensure(nwy * sizeof(float))) CTK_CUDA(cudaMemsetAsync(wy.p, 0, nwy * sizeof(float), s));
    dim3 blk(32, 8), grd((g.nx + 31) / 32, (g.nz_local() + 31) / 32, g.ny);
    k_relayout_zfast<<<grd, blk, 0, s>>>(g.nx, g.ny, g.nz_local(), x, wx.as<float>(), wy.as<float>());
    after_launch("k_relayout_zfast");
}

dim3 fwd_grid(const Geometry& g) { return dim3((g.nu + ZW_BC - 1) / ZW_BC, g.na, (g.nv + ZW_BR - 1) / ZW_BR); }

// 64-bit tap offsets once a padded layout exceeds 2^31 elements (volumes beyond ~1290^3);
// CTK_FWD_WIDE=1 forces them (tests exercise that instantiation on small volumes)
bool wide_offsets(const Geometry& g) {
    static const bool forced = [] {
        const char* e = std::getenv("CTK_FWD_WIDE");
        return e && e[0] == '1';
    }();
    const double mx = std::max(double(g.nx) * (g.ny + 2 * kPad), double(g.ny) * (g.nx + 2 * kPad)) * (g.nz_local() + 2 * kPad);
    return forced || mx >= 2147483000.0;
}

template <int MODE>
void launch_ax(Geometry& g, const float* x, float* y, const float* b, double* partials, cudaStream_t s, int nch = 1,
               int chunk = 0, int band0 = 0, int band1 = -1) {
    const KGeom k = g.kgeom();
    const int* vo = g.d_vorder.as<int>();
    const float *a0 = g.vx.as<float>(), *a1 = g.vy.as<float>();
    const dim3 blk(ZW_BR, ZW_BC);
    dim3 grd = fwd_grid(g);
    if (band1 >= 0) grd.z = unsigned(band1 - band0);
    if (grd.z == 0) return;
    const bool sid = g.projector == CTK_PROJ_SIDDON;  // (no band-sharded range with Siddon)
    if (wide_offsets(g)) {
        if (sid) k_ax_zfast_f32<MODE, long long, 1><<<grd, blk, 0, s>>>(k, vo, a0, a1, x, y, b, partials, nch, chunk, band0);
        else if (g.band) k_ax_zfast_f32<MODE, long long, 0, 1><<<grd, blk, 0, s>>>(k, vo, a0, a1, x, y, b, partials, nch, chunk, band0);
        else k_ax_zfast_f32<MODE, long long><<<grd, blk, 0, s>>>(k, vo, a0, a1, x, y, b, partials, nch, chunk, band0);
    } else {
        if (sid) k_ax_zfast_f32<MODE, int, 1><<<grd, blk, 0, s>>>(k, vo, a0, a1, x, y, b, partials, nch, chunk, band0);
        else if (g.band) k_ax_zfast_f32<MODE, int, 0, 1><<<grd, blk, 0, s>>>(k, vo, a0, a1, x, y, b, partials, nch, chunk, band0);
        else k_ax_zfast_f32<MODE, int><<<grd, blk, 0, s>>>(k, vo, a0, a1, x, y, b, partials, nch, chunk, band0);
    }
    after_launch(MODE == 0 ? "k_ax_zfast_f32" : "k_ax_zfast_f32_residual");
}

// Slice chunks per ray: enough that the slab a (row band, chunk) pass touches -- about
// 200 B per (slice, in-plane row) for a 32-row band -- stays near 26 MB, i.e. L2-resident
// across all views; at least 2 (measured: 2 at 256^3 and 512^3, 8 at 1024^3: 3.06 s with 2
// chunks vs 1.70 s with 8).  CTK_FWD_CHUNKS (environment) overrides.
int fwd_chunks(const Geometry& g) {
    static const int forced = [] {
        const char* e = std::getenv("CTK_FWD_CHUNKS");
        return e ? std::max(1, std::atoi(e)) : 0;
    }();
    if (forced) return forced;
    const double slab = double(std::max(g.nx, g.ny)) * (std::max(g.nx, g.ny) + 2) * 200.0;
    const int base = std::max(CTK_FWD_CHUNKS, std::min(16, int(std::lround(slab / 26e6))));
    // fewer views per handle (an angle-sharded rank) -> fewer reuses of each slab: halve it
    // (512^3: 45/90/180 views 7.43/13.57/25.33 -> 7.03/13.02/24.88 ms with 4 chunks, 360 views
    // unchanged; at 256^3 the minimum of 2 stays best at every view count)
    return (g.na < 300 && slab > 26e6) ? std::min(16, 2 * base) : base;
}

// Detector-row bands whose rays can reach this handle's slices.  A cone ray through row
// coordinate v meets height z at depth d (from the source) where z = v d / (DSO + DOD), and
// the volume spans depths DSO -+ R (R: in-plane half-diagonal), so a z-slab is seen only by
// the rows between its edges' images at the nearest and farthest depth (parallel beams:
// v = z).  With a thin slab most bands see nothing: they are not launched (their rows are
// zeroed instead).  Whole-volume handles keep every band.
void slab_bands(const Geometry& g, int& b0, int& b1) {
    const int nb = (g.nv + ZW_BR - 1) / ZW_BR;
    b0 = 0;
    b1 = nb;
    if (!g.slab || g.nv == 1) return;
    int r0, r1;
    slab_rows(g, g.z0, g.nz_local(), r0, r1);
    if (g.band) {  // only the rows this rank holds
        r0 = std::max(r0, g.w0);
        r1 = std::min(r1, g.w0 + g.nw);
    }
    if (r1 <= r0) {
        b1 = b0;
        return;
    }
    b0 = r0 / ZW_BR;
    b1 = std::min(nb, (r1 + ZW_BR - 1) / ZW_BR);
}

double* residual_partials(Geometry& g, size_t& nblk) {
    const dim3 grd = fwd_grid(g);
    nblk = size_t(grd.x) * grd.y * grd.z;
    g.proj_t.ensure(std::max(g.range() * sizeof(float), nblk * sizeof(double)));
    return g.proj_t.as<double>();
}

}  // namespace

void ax_f32(Geometry& g, const float* x, float* y, cudaStream_t s) {
    relayout_zfast(g, x, g.vx, g.vy, s);
    const int nch = fwd_chunks(g);
    int b0, b1;
    slab_bands(g, b0, b1);
    CTK_CUDA(cudaEventRecord(g.ev0, s));
    if (b0 > 0 || b1 < int((g.nv + ZW_BR - 1) / ZW_BR) || g.band)
        CTK_CUDA(cudaMemsetAsync(y, 0, g.range() * sizeof(float), s));  // rows no launched band writes
    for (int c = 0; c < nch; ++c) launch_ax<0>(g, x, y, nullptr, nullptr, s, nch, c, b0, b1);
    CTK_CUDA(cudaEventRecord(g.ev1, s));
    // Siddon: the z-dominant rays take the exact DDA (siddon.cu), writing only their entries
    if (g.projector == CTK_PROJ_SIDDON && g.has_zrays) siddon_ax_zrays_f32(g, x, y, s);
}

bool ax2_f32_supported(const Geometry& g) {
    const char* e = std::getenv("CTK_FWD_NO_PAIR");  // read per call: tests switch it in-process
    // whole volume: no slab, or a slab handle that holds every slice (a one-rank z-slab run)
    const bool whole = !g.slab || (g.z0 == 0 && g.nz_local() == g.nz);
    return !(e && e[0] == '1') && whole && !g.band;
}

void ax2_f32(Geometry& g, const float* x1, float* y1, const float* x2, float* y2, cudaStream_t s) {
    if (!ax2_f32_supported(g)) throw Error(CTK_E_UNSUPPORTED, "ax2_f32: whole-volume handles only");
    const size_t nwx = size_t(g.nx) * (size_t(g.ny) + 2 * kPad) * (size_t(g.nz) + 2 * kPad);
    const size_t nwy = size_t(g.ny) * (size_t(g.nx) + 2 * kPad) * (size_t(g.nz) + 2 * kPad);
    if (g.vx2.ensure(nwx * sizeof(float2))) CTK_CUDA(cudaMemsetAsync(g.vx2.p, 0, nwx * sizeof(float2), s));
    if (g.vy2.ensure(nwy * sizeof(float2))) CTK_CUDA(cudaMemsetAsync(g.vy2.p, 0, nwy * sizeof(float2), s));
    {
        dim3 blk(32, 8), grd((g.nx + 31) / 32, (g.nz + 31) / 32, g.ny);
        k_relayout2_zfast<<<grd, blk, 0, s>>>(g.nx, g.ny, g.nz, x1, x2, g.vx2.as<float2>(), g.vy2.as<float2>());
        after_launch("k_relayout2_zfast");
    }
    const int nch = fwd_chunks(g);  // as ax_f32: the chunk sums must match for bit-identical outputs
    const KGeom k = g.kgeom();
    const int* vo = g.d_vorder.as<int>();
    const float2 *a0 = g.vx2.as<float2>(), *a1 = g.vy2.as<float2>();
    const dim3 blk(ZW_BR, ZW_BC), grd = fwd_grid(g);
    CTK_CUDA(cudaEventRecord(g.ev0, s));
    // 64-bit offsets once the float2 layout's element count passes 2^31 (offsets index float2)
    for (int c = 0; c < nch; ++c) {
        const bool sid = g.projector == CTK_PROJ_SIDDON;
        if (wide_offsets(g)) {
            if (sid) k_ax2_zfast_f32<long long, 1><<<grd, blk, 0, s>>>(k, vo, a0, a1, x1, x2, y1, y2, nch, c);
            else k_ax2_zfast_f32<long long, 0><<<grd, blk, 0, s>>>(k, vo, a0, a1, x1, x2, y1, y2, nch, c);
        } else {
            if (sid) k_ax2_zfast_f32<int, 1><<<grd, blk, 0, s>>>(k, vo, a0, a1, x1, x2, y1, y2, nch, c);
            else k_ax2_zfast_f32<int, 0><<<grd, blk, 0, s>>>(k, vo, a0, a1, x1, x2, y1, y2, nch, c);
        }
        after_launch("k_ax2_zfast_f32");
    }
    CTK_CUDA(cudaEventRecord(g.ev1, s));
    // Siddon: the z-dominant rays by the exact DDA, writing only their entries (as ax_f32)
    if (g.projector == CTK_PROJ_SIDDON && g.has_zrays) {
        siddon_ax_zrays_f32(g, x1, y1, s);
        siddon_ax_zrays_f32(g, x2, y2, s);
    }
}

void ax_residual_f32(Geometry& g, const float* x, const float* b, double* d_out, cudaStream_t s) {
    if (fwd_chunks(g) > 1 || g.projector == CTK_PROJ_SIDDON) {  // chunked: A x into a scratch projection set, then the fused difference norm
        g.ax_scratch.ensure(g.range() * sizeof(float));
        ax_f32(g, x, g.ax_scratch.as<float>(), s);
        RedWork w = red_work(&g);
        reduce_diff_nrm2sq<float>(g.range(), g.ax_scratch.as<float>(), b, d_out, w, s);
        return;
    }
    relayout_zfast(g, x, g.vx, g.vy, s);
    size_t nblk;
    double* partials = residual_partials(g, nblk);
    CTK_CUDA(cudaEventRecord(g.ev0, s));
    launch_ax<1>(g, x, nullptr, b, partials, s);
    CTK_CUDA(cudaEventRecord(g.ev1, s));
    finish_sum(partials, int(nblk), d_out, s);
}

}  // namespace ctkb
