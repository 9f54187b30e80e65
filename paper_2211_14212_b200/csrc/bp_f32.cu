// A^T b for T = float on sm_100a: the exact transpose of fwd_f32.cu (matched) and the
// voxel-driven backprojection (projector.hpp:204-279).  Both gather -- the matched one from
// the step-scaled projections in 4-row groups pg[a][iv/4][iu][iv%4], the voxel-driven one
// from the projections transposed to pt[a][iu][iv] -- so no float atomics are used and
// every voxel sums its contributions in a fixed order.
#include <cstdlib>
#include <mutex>

#include "f32_common.cuh"

namespace ctkb {
namespace {

// ---- projection transpose for the gathers: pt[a][iu][iv] = (step?) * y[a][iv][iu] ------
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
            pt[(size_t(a) * g.nu + iu) * g.nv + iv] = tile[threadIdx.x][r];
        }
    }
}

// ---- grouped projection layout for the matched gather: pg[a][iv/4][iu][iv%4] = step * y ----
// A warp of the plane kernel = 32 consecutive detector columns marching their rows in 4-row
// groups (one 16-byte load per lane): with the columns of a row group contiguous, the warp's
// load is one contiguous 512-byte run instead of 32 scattered 16-byte pieces.  Rows are
// zero-padded to a multiple of 4.
// row groups per view, rounded up to even so the plane kernel can march whole pairs of groups
// (the padding groups are zero)
__host__ __device__ __forceinline__ int pg_groups(int nv) { return (((nv + 3) >> 2) + 1) & ~1; }
__device__ __forceinline__ size_t pg_index(const KGeom& g, int a, int iu, int iv) {
    return ((size_t(a) * pg_groups(g.nv) + (iv >> 2)) * g.nu + iu) * 4 + (iv & 3);
}

__global__ void k_proj_group4(KGeom g, const float* __restrict__ y, float* __restrict__ pg) {
    // block: 32 columns x 8 row groups; thread (u, q) writes one float4
    const int a = blockIdx.z;
    const int iu = blockIdx.x * 32 + threadIdx.x, q = blockIdx.y * 8 + threadIdx.y;
    const int nq = pg_groups(g.nv);
    if (iu >= g.nu || q >= nq) return;
    const int c = a * g.nu + iu;
    const double2 cs = g.colstep[c];
    const float* fr = y + size_t(a) * g.nu * g.nv;
    float r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int iv = 4 * q + j;
        r[j] = iv < g.nv ? __ldg(fr + size_t(iv) * g.nu + iu) * ray_step(g, cs, row_coord(g, iv)) : 0.f;
    }
    reinterpret_cast<float4*>(pg)[(size_t(a) * nq + q) * g.nu + iu] = make_float4(r[0], r[1], r[2], r[3]);
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
// Tile size PB (rows = threads per CTA) is a template parameter with its own row-list
// capacity SL and occupancy (measured, matched A^T b f32):
//   PB = 128, 6 CTAs/SM: 256^3/180 4.61 ms, 512^3/360 66.9 ms (SL = 9/10/11/12: 71.2/67.7/66.9/69.0)
//   PB = 256, 3 CTAs/SM: 256^3/180 5.32 ms, 512^3/360 72.8 ms, 512^3/720 147 ms,
//                        1024^3/1600 2518 ms at SL = 11 (SL = 10/12/14: 2563/2565/3275;
//                        PB = 128: 3034 ms -- per-CTA setup over 1600 views, twice the tiles)
// so the launcher takes PB = 128 up to 768 rows per plane and PB = 256 beyond.  Smaller
// lists (SL = 8 at PB = 128) overflow into the slow scan: 74.5 ms.  Without view batching
// 4 CTAs/SM (64 regs) was best.
#ifndef CTK_BP_SL128
#define CTK_BP_SL128 11
#endif
#ifndef CTK_BP_SL256
#define CTK_BP_SL256 11
#endif
// Phase 2 by row PAIRS (CTK_BP_PAIR=1): thread = (row pair, half of the z band).  A column
// registered in rows ih and ih+1 with ih even feeds BOTH rows of one pair from a single read
// of its Z column (one FFMA2 per slice on the packed (row 2r, row 2r+1) accumulators), so
// the shared-memory reads of phase 2 drop from ~2 to ~1.5 per (column, row) registration.
#ifndef CTK_BP_PAIR
#define CTK_BP_PAIR 0
#endif
#ifndef CTK_BP_SL2
#define CTK_BP_SL2 14
#endif
#ifndef CTK_BP_TIGHT
#define CTK_BP_TIGHT 0
#endif
template <int PB>
struct PlaneCfg;
template <>
struct PlaneCfg<128> {
    static constexpr int SL = CTK_BP_PAIR ? CTK_BP_SL2 : CTK_BP_SL128, MINB = 6;
};
template <>
struct PlaneCfg<256> {
    static constexpr int SL = CTK_BP_PAIR ? CTK_BP_SL2 : CTK_BP_SL256, MINB = 3;
};
#ifndef CTK_BP_KB
#define CTK_BP_KB 32
#endif
constexpr int BP_KB = CTK_BP_KB;
constexpr int BP_ZG = 2;
// Z column swizzle (CTK_BP_SWZ=1): slot e lives in column e + e/32 of a row of stride
// PB + PB/32, so slots e and e+32 fall in different banks.  Phase-2 lanes (consecutive rows
// or row pairs) read slots about one or two apart, which without it pairs lanes l and l+16
// on one bank whenever the slots span more than 32; phase-1 lanes (32 consecutive slots)
// stay conflict-free.
#ifndef CTK_BP_SWZ
#define CTK_BP_SWZ 0
#endif
template <int PB>
__host__ __device__ constexpr int z_stride() { return PB + (CTK_BP_SWZ ? PB / 32 : 0); }
__device__ __forceinline__ int z_col(int e) { return CTK_BP_SWZ ? e + (e >> 5) : e; }
  // guard rows of Z on each side: out-of-band entries land there, unread

template <int CLASS, int PB>
__global__ void __launch_bounds__(PB, PlaneCfg<PB>::MINB)
k_atb_plane_f32(KGeom g, const float* __restrict__ pg, float* __restrict__ x, int ptiles) {
    constexpr int BP_PB = PB, BP_SL = PlaneCfg<PB>::SL;
    constexpr int NL = CTK_BP_PAIR ? PB / 2 : PB;  // registration lists: per row pair / per row
    extern __shared__ __align__(16) float sm[];
    constexpr int ZS = z_stride<PB>();                          // row stride of Z
    float* Z = sm + BP_ZG * ZS;                                 // [-BP_ZG, BP_KB+BP_ZG) x [ZS]
    int* lists = reinterpret_cast<int*>(Z + (BP_KB + BP_ZG) * ZS);  // [NL][BP_SL]
    int* cnt = lists + NL * BP_SL;                              // [NL]
    float* eth = reinterpret_cast<float*>(cnt + NL);            // [BP_PB]
    static_assert((NL * BP_SL) % 4 == 0 && NL % 4 == 0, "keeps vrtab 16-byte aligned");
    const int nv4 = 4 * pg_groups(g.nv);
    float* vrtab = eth + BP_PB;                                 // [nv4] iv - (nv-1)/2, 16-byte aligned
    int2* urange = reinterpret_cast<int2*>(vrtab + nv4);        // [na]
    int* pref = reinterpret_cast<int*>(urange + g.na);          // [na + 1] candidate prefix sums
    int* slotcol = pref + g.na + 1;                             // [BP_PB] (view, column) of a slot

    const int t = threadIdx.x;
    // plane index fastest: a wave of resident CTAs shares one (row tile, z band), so per
    // view it reads only that band's detector rows -> the projections stay L2-resident
    const int s = blockIdx.x;
    const int ptile = blockIdx.y % ptiles, kband = blockIdx.y / ptiles;
    const int p0 = ptile * BP_PB, k0 = kband * BP_KB;
    const int nh = CLASS ? g.nx : g.ny;
    const int p = p0 + t;
    for (int q = t; q < nv4; q += BP_PB) vrtab[q] = row_vr(g, q);
    const int sc = slice_centre(s);  // anchored positions (f32_common.cuh): block centre of plane s
    const float kf = float(s - sc);
    const float czf = 0.5f * float(g.nzg - 1);  // global z centre; this handle's slices start at z0
    const int kg0 = k0 + g.z0;                   // global index of the band's first slice
    const float cvf = 0.5f * float(g.nv - 1);
    const float invdu = float(1.0 / g.du);
    const float fs = float(s);
    const double h = g.h;
    const int nq = pg_groups(g.nv);  // row groups of the grouped projection layout
    // world coordinates of the plane and of the tile's row segment ends
    const double plane_c = (s - 0.5 * ((CLASS ? g.ny : g.nx) - 1)) * h;
    const double r_lo = (p0 - 1.5 - 0.5 * (nh - 1)) * h, r_hi = (p0 + BP_PB + 0.5 - 0.5 * (nh - 1)) * h;

#if CTK_BP_PAIR
    // thread = (row pair r: rows p0+2r, p0+2r+1; half kh of the z band): BP_KB/2 packed
    // accumulators (row 2r, row 2r+1) per slice
    const int r2 = t % (BP_PB / 2), kh = t / (BP_PB / 2);
    const int kz0 = kh * (BP_KB / 2);
    float2 acc2[BP_KB / 2];
#pragma unroll
    for (int m = 0; m < BP_KB / 2; ++m) acc2[m] = make_float2(0.f, 0.f);
    auto add_entry2 = [&](float2 w2, int e) {
        const int ze = z_col(e);
#pragma unroll
        for (int m = 0; m < BP_KB / 2; ++m) {
            const float z = Z[(kz0 + m) * ZS + ze];
            acc2[m] = __ffma2_rn(w2, make_float2(z, z), acc2[m]);
        }
    };
#else
    // BP_KB accumulators as packed pairs: phase 2 adds wh * Z with FFMA2 (per element the
    // scalar fma)
    float2 acc2[BP_KB / 2];
#pragma unroll
    for (int m = 0; m < BP_KB / 2; ++m) acc2[m] = make_float2(0.f, 0.f);
    auto add_entry = [&](float wh, int e) {
        const float2 w2 = make_float2(wh, wh);
        const int ze = z_col(e);
#pragma unroll
        for (int m = 0; m < BP_KB / 2; ++m)
            acc2[m] = __ffma2_rn(w2, make_float2(Z[(2 * m) * ZS + ze], Z[(2 * m + 1) * ZS + ze]), acc2[m]);
    };
#endif

    // candidate detector-column range of every view for this tile (projection of the
    // tile's row segment in the plane), computed once, in parallel
    for (int a = t; a < g.na; a += BP_PB) {
        const double2 tr = g.ctst[a];
        bool ok1, ok2;
        const double u1 = CLASS ? proj_u(g, tr.x, tr.y, r_lo, plane_c, ok1) : proj_u(g, tr.x, tr.y, plane_c, r_lo, ok1);
        const double u2 = CLASS ? proj_u(g, tr.x, tr.y, r_hi, plane_c, ok2) : proj_u(g, tr.x, tr.y, plane_c, r_hi, ok2);
        int i0 = 0, i1 = g.nu - 1;
        if (ok1 && ok2) {
            i0 = max(i0, int(floor(fmax(fmin(u1, u2), -1e9))) - 1);
            i1 = min(i1, int(ceil(fmin(fmax(u1, u2), 1e9))) + 1);
        }
        // only this pass's ray class: intersect with the hull of the view's CLASS columns
        const int4 vc = g.vclass[a];
        i0 = max(i0, CLASS ? vc.z : vc.x);
        i1 = min(i1, CLASS ? vc.w : vc.y);
        urange[a] = make_int2(i0, i1);
    }
    __syncthreads();
    // Candidate (view, column) pairs of all views are packed into batches of BP_PB slots
    // (view-major, columns ascending), so a batch mixes the tail of one view with the head
    // of the next and no thread idles on a half-empty chunk.  Per voxel the summation order
    // is unchanged: entries are still added in (view, column) order.
    if (t < 32) {  // exclusive prefix sum of the candidate counts, one warp
        int run = 0;
        for (int a0 = 0; a0 < g.na; a0 += 32) {
            const int a = a0 + t;
            const int n = a < g.na ? max(0, urange[a].y - urange[a].x + 1) : 0;
            int incl = n;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int o = __shfl_up_sync(0xffffffffu, incl, d);
                if (t >= d) incl += o;
            }
            if (a < g.na) pref[a] = run + incl - n;
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (t == 0) pref[g.na] = run;
    }
    __syncthreads();
    const int total = pref[g.na];
    int a_run = 0;  // this thread's slot view, advanced monotonically across batches

    for (int b0 = 0; b0 < total; b0 += BP_PB) {
        {
            // ---- phase 1 ----
            if (t < NL) cnt[t] = 0;
            int a = -1, iu = 0;
            const int gidx = b0 + t;
            if (gidx < total) {  // the view of this slot: pref[a] <= gidx < pref[a + 1]
                while (pref[a_run + 1] <= gidx) ++a_run;  // monotone over batches: ~1 step
                a = a_run;
                iu = urange[a].x + (gidx - pref[a]);
            }
            slotcol[t] = a >= 0 ? a * g.nu + iu : -1;
            __syncthreads();
            if (a >= 0) {
                const int c = a * g.nu + iu;
                if (g.colaxis[c] == CLASS) {
                    const float4 cd = g.col[c];
                    const double4 c64 = g.col64[c];
                    int ih, ihA;
                    float th, thA;
                    double G;
                    slice_anchor(c64, sc, ihA, thA, G);  // fh exactly as the forward evaluates it
                    split(fmaf(kf, cd.y, thA), ih, th);
                    ih += ihA;
                    if (ih + 1 >= p0 && ih <= p0 + BP_PB - 1 && ih + 1 >= 0 && ih < nh) {
                        const float gs = fmaf(fs, cd.w, cd.z);
                        int v0 = 0, v1 = g.nv - 1;
                        if (gs > 0.f) {
                            const float rg = invdu / gs;
                            v0 = max(v0, int(floorf(fmaf(float(kg0) - 1.f - czf, rg, cvf))) - 1);
                            v1 = min(v1, int(ceilf(fmaf(float(kg0 + BP_KB) - czf, rg, cvf))) + 1);
                        }
                        if (g.has_zrays) {
                            // rows whose ray is z-dominant (|v| > |d_A|) belong to the generic
                            // pass; they form the two ends of the column: clip exactly
                            const double dA = g.colstep[c].y;
                            const double cv = 0.5 * (g.nv - 1), r = dA / g.du;
                            int lo = max(v0, int(ceil(cv - r)) - 1), hi = min(v1, int(floor(cv + r)) + 1);
                            while (lo <= hi && fabs(row_coord(g, lo)) > dA) ++lo;
                            while (hi >= lo && fabs(row_coord(g, hi)) > dA) --hi;
                            v0 = lo;
                            v1 = hi;
                        }
                        // column iu of view a, row group q: pc4[q * nu] (grouped layout)
                        const float4* pc4 = reinterpret_cast<const float4*>(pg) + size_t(a) * nq * g.nu + iu;
                        const size_t qs = size_t(g.nu);
                        float* zc = Z + z_col(t);
                        // z of row iv at this plane (f32_common.cuh), the forward's expression:
                        //   S = fmaf(vr, Whi, fc) (exact), T = fmaf(vr, Wlo, S),
                        //   iz = izc + floor(T), tz = fmaf(vr, Wlo, S - floor(T))
                        float Whi, Wr;
                        z_split(g, G, Whi, Wr);
                        const float Wlo = fmaf(kf, z_cross(g, c64), Wr), fc = cz_frac(g);
                        const int koff = cz_int(g) - kSplitBias - kg0;  // kk = bits(T + M, rd) + koff
                        float tf_unused;
                        auto row_k = [&](int iv, float& tz) {  // band slice index of row iv's z floor
                            const float vr = vrtab[iv];
                            const float S = fmaf(vr, Whi, fc);
                            const float tt = split_t(fmaf(vr, Wlo, S));
                            tz = fmaf(vr, Wlo, fmaf(__fsub_rn(tt, kSplitM), -1.f, S));
                            return __float_as_int(tt) + koff;
                        };
                        auto zero_rows = [&](int lo, int hi) {  // Z rows [lo, hi) of this column
                            for (int m = max(lo, 0); m < min(hi, BP_KB); ++m) zc[m * ZS] = 0.f;
                        };
                        if (gs > 0.f && v0 <= v1) {
                            // fz increases with iv, so Z[k] is final once the march passes it:
                            // accumulate in registers (A -> Z[cur], B -> Z[cur+1]) and store both
                            // after every row, unconditionally (a later row either overwrites them
                            // with a larger partial or has moved past; measured faster than
                            // predicated once-only stores, which compile to branches).
                            // Out-of-band k land in the guard rows.  With at least 0.75 rows per
                            // slice fz advances < 1.34 per row, so k never skips an entry and
                            // only the rows before the first / after the last k need zeroing;
                            // sparser columns zero the whole band first.
                            const float rg = invdu / gs;
#if CTK_BP_TIGHT
                            // trim the estimated row range to the rows whose z stencil meets the
                            // band (kk in [-1, BP_KB-1]), with the exact arithmetic of the march:
                            // rows outside only reach the guard rows
                            while (v0 < v1 && row_k(v0, tf_unused) < -1) ++v0;
                            while (v1 > v0 && row_k(v1, tf_unused) > BP_KB - 1) --v1;
#endif
                            if (rg >= 0.75f) {
                                zero_rows(0, row_k(v0, tf_unused));
                            } else {
                                zero_rows(0, BP_KB);
                            }
                            int cur = -(1 << 20);
                            float A = 0.f, B = 0.f;
                            // one row: tt = fz + 1.5*2^23 rounded down (its bits carry the slice
                            // index), tz = the z fraction, omt = 1 - tz
                            auto step_w = [&](int kk, float tz, float omt, float yv) {
                                const float w0 = omt * yv, w1 = tz * yv;
                                const int adv = kk - cur;
                                float ak = adv == 1 ? B : 0.f;  // two selects, no branch
                                ak = adv == 0 ? A : ak;
                                const float bk = adv == 0 ? B : 0.f;
                                A = ak + w0;
                                B = bk + w1;
                                cur = kk;
                                // one unsigned clamp: kk < -BP_ZG wraps high and lands in the top guard rows
                                float* zp = zc - BP_ZG * ZS + min(unsigned(kk + BP_ZG), unsigned(BP_KB + 2 * BP_ZG - 2)) * ZS;
                                zp[0] = A;
                                zp[ZS] = B;
                            };
                            // the row positions of a 4-row group in packed f32x2 arithmetic
                            // (FFMA2 / FADD2), per lane the scalar sequence of row_k
                            const float2 Whi2 = make_float2(Whi, Whi), Wlo2 = make_float2(Wlo, Wlo), fc2 = make_float2(fc, fc);
                            const float2 M2 = make_float2(kSplitM, kSplitM), nM2 = make_float2(-kSplitM, -kSplitM);
                            const float2 m1 = make_float2(-1.f, -1.f), one2 = make_float2(1.f, 1.f);
                            auto step2 = [&](float2 vr, float ya, float yb) {
                                const float2 S = __ffma2_rn(vr, Whi2, fc2);
                                const float2 tt = __fadd2_rd(__ffma2_rn(vr, Wlo2, S), M2);
                                const float2 tz = __ffma2_rn(vr, Wlo2, __ffma2_rn(__fadd2_rn(tt, nM2), m1, S));
                                const float2 omt = __ffma2_rn(tz, m1, one2);
                                step_w(__float_as_int(tt.x) + koff, tz.x, omt.x, ya);
                                step_w(__float_as_int(tt.y) + koff, tz.y, omt.y, yb);
                            };
                            // whole 4-row groups; only the first and last are masked to [v0, v1]
                            const float4* vr4 = reinterpret_cast<const float4*>(vrtab);
                            const int q0 = v0 >> 2, q1 = v1 >> 2;
                            CTK_CHK(g, q0 >= 0 && q1 < nq && size_t(a) < size_t(g.na) && iu < g.nu, 1);
                            auto group = [&](int q, float4 y4, bool mask) {
                                const float4 d4 = vr4[q];
                                if (mask) {
                                    const int b = 4 * q;
                                    y4.x = (b >= v0 && b <= v1) ? y4.x : 0.f;
                                    y4.y = (b + 1 >= v0 && b + 1 <= v1) ? y4.y : 0.f;
                                    y4.z = (b + 2 >= v0 && b + 2 <= v1) ? y4.z : 0.f;
                                    y4.w = (b + 3 >= v0 && b + 3 <= v1) ? y4.w : 0.f;
                                }
                                step2(make_float2(d4.x, d4.y), y4.x, y4.y);
                                step2(make_float2(d4.z, d4.w), y4.z, y4.w);
                            };
                            // two row groups per iteration: two 16-byte loads in flight
                            group(q0, __ldg(pc4 + q0 * qs), true);
                            int q = q0 + 1;
                            for (; q + 1 < q1; q += 2) {
                                const float4 ya = __ldg(pc4 + q * qs), yb = __ldg(pc4 + (q + 1) * qs);
                                group(q, ya, false);
                                group(q + 1, yb, false);
                            }
                            if (q < q1) group(q, __ldg(pc4 + q * qs), false);
                            if (q1 > q0) group(q1, __ldg(pc4 + q1 * qs), true);
                            zero_rows(cur + 2, BP_KB);
                        } else {
                            // no rows, or degenerate geometry (stencil point not in front of the source)
                            zero_rows(0, BP_KB);
                            for (int iv = v0; iv <= v1; ++iv) {
                                const float yv = reinterpret_cast<const float*>(pc4 + (iv >> 2) * qs)[iv & 3];
                                float tz;
                                const int kk = row_k(iv, tz);
                                if (unsigned(kk) < unsigned(BP_KB)) zc[kk * ZS] = fmaf(1.f - tz, yv, zc[kk * ZS]);
                                if (unsigned(kk + 1) < unsigned(BP_KB)) zc[(kk + 1) * ZS] = fmaf(tz, yv, zc[(kk + 1) * ZS]);
                            }
                        }
                        eth[t] = th;
#if CTK_BP_PAIR
                        // rows rel (weight 1-th) and rel+1 (weight th), relative to p0 (even):
                        // mode 0 = both rows of pair rel/2, 1 = row rel as the .y of its pair,
                        // 2 = row rel+1 as the .x of its pair
                        auto reg = [&](int pr, int mode) {
                            const int sl = atomicAdd(&cnt[pr], 1);
                            if (sl < BP_SL) lists[pr * BP_SL + sl] = (t << 2) | mode;
                        };
                        const int rel = ih - p0;
                        if (!(rel & 1)) {
                            reg(rel >> 1, 0);
                        } else {
                            if (rel >= 0) reg(rel >> 1, 1);
                            if (rel + 1 <= BP_PB - 1 && th != 0.f) reg((rel + 1) >> 1, 2);
                        }
#else
                        if (ih >= p0) {
                            const int sl = atomicAdd(&cnt[ih - p0], 1);
                            if (sl < BP_SL) lists[(ih - p0) * BP_SL + sl] = (t << 1);
                        }
                        if (ih + 1 <= p0 + BP_PB - 1 && th != 0.f) {
                            const int sl = atomicAdd(&cnt[ih + 1 - p0], 1);
                            if (sl < BP_SL) lists[(ih + 1 - p0) * BP_SL + sl] = (t << 1) | 1;
                        }
#endif
                    }
                }
            }
            __syncthreads();
#if CTK_BP_PAIR
            // ---- phase 2: row pair r2 gathers its registered columns in column order ----
            const int n = cnt[r2];
            if (n > 0 && p0 + 2 * r2 < nh) {
                if (n <= BP_SL) {
                    int lst[BP_SL];
#pragma unroll
                    for (int q = 0; q < BP_SL; ++q) lst[q] = q < n ? lists[r2 * BP_SL + q] : 0x7fffffff;
                    // insertion sort of the n registered entries (n is small: 3-6 typically)
#pragma unroll
                    for (int i = 1; i < BP_SL; ++i) {
                        if (i >= n) break;
#pragma unroll
                        for (int j = i; j > 0; --j)
                            if (lst[j - 1] > lst[j]) { const int tmp = lst[j]; lst[j] = lst[j - 1]; lst[j - 1] = tmp; }
                    }
#pragma unroll
                    for (int q = 0; q < BP_SL; ++q) {
                        if (q >= n) break;
                        const int e = lst[q] >> 2, mode = lst[q] & 3;
                        const float th = eth[e], omt = 1.f - th;
                        const float2 w2 = mode == 0 ? make_float2(omt, th) : (mode == 1 ? make_float2(0.f, omt) : make_float2(th, 0.f));
                        add_entry2(w2, e);
                    }
                } else {
                    // overflow (very fine detector sampling): scan every slot of the batch in order
                    const int pa = p0 + 2 * r2;
                    for (int e = 0; e < BP_PB; ++e) {
                        const int c = slotcol[e];
                        if (c < 0 || g.colaxis[c] != CLASS) continue;
                        int ih, ihA;
                        float th, thA;
                        double G;
                        slice_anchor(g.col64[c], sc, ihA, thA, G);
                        split(fmaf(kf, g.col[c].y, thA), ih, th);
                        ih += ihA;
                        if (ih + 1 < p0 || ih > p0 + BP_PB - 1 || ih + 1 < 0 || ih >= nh) continue;  // not registered
                        const float omt = 1.f - th;
                        float2 w2;
                        if (ih == pa) w2 = make_float2(omt, th);
                        else if (ih == pa + 1) w2 = make_float2(0.f, omt);
                        else if (ih + 1 == pa && th != 0.f) w2 = make_float2(th, 0.f);
                        else continue;
                        add_entry2(w2, e);
                    }
                }
            }
#else
            // ---- phase 2: row p gathers its registered columns in column order ----
            const int n = cnt[t];
            if (n > 0 && p < nh) {
                if (n <= BP_SL) {
                    int lst[BP_SL];
#pragma unroll
                    for (int q = 0; q < BP_SL; ++q) lst[q] = q < n ? lists[t * BP_SL + q] : 0x7fffffff;
                    // insertion sort of the n registered entries (n is small: 2-6 typically)
#pragma unroll
                    for (int i = 1; i < BP_SL; ++i) {
                        if (i >= n) break;
#pragma unroll
                        for (int j = i; j > 0; --j)
                            if (lst[j - 1] > lst[j]) { const int tmp = lst[j]; lst[j] = lst[j - 1]; lst[j - 1] = tmp; }
                    }
#pragma unroll
                    for (int q = 0; q < BP_SL; ++q) {
                        if (q >= n) break;
                        const int e = lst[q] >> 1;
                        CTK_CHK(g, e < BP_PB, 3);
                        const float th = eth[e];
                        const float wh = (lst[q] & 1) ? th : 1.f - th;
                        add_entry(wh, e);
                    }
                } else {
                    // overflow (very fine detector sampling): scan every slot of the batch in order
                    for (int e = 0; e < BP_PB; ++e) {
                        const int c = slotcol[e];
                        if (c < 0 || g.colaxis[c] != CLASS) continue;
                        int ih, ihA;
                        float th, thA;
                        double G;
                        slice_anchor(g.col64[c], sc, ihA, thA, G);
                        split(fmaf(kf, g.col[c].y, thA), ih, th);
                        ih += ihA;
                        float wh;
                        if (ih == p) wh = 1.f - th;
                        else if (ih + 1 == p && th != 0.f) wh = th;
                        else continue;
                        add_entry(wh, e);
                    }
                }
            }
#endif
            __syncthreads();
        }
    }
#if CTK_BP_PAIR
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
        const int pr = p0 + 2 * r2 + h2;
        if (pr >= nh) break;
#pragma unroll
        for (int m = 0; m < BP_KB / 2; ++m) {
            const int k = k0 + kz0 + m;
            if (k >= g.nz) break;
            const size_t o = CLASS ? size_t(pr) + size_t(g.nx) * (size_t(s) + size_t(g.ny) * k)
                                   : size_t(s) + size_t(g.nx) * (size_t(pr) + size_t(g.ny) * k);
            const float am = h2 ? acc2[m].y : acc2[m].x;
            if (CLASS == 0) x[o] = am;
            else x[o] += am;
        }
    }
#else
    if (p < nh) {
#pragma unroll
        for (int m = 0; m < BP_KB; ++m) {
            const int k = k0 + m;
            if (k >= g.nz) break;
            const size_t o = chk_idx(g, CLASS ? size_t(p) + size_t(g.nx) * (size_t(s) + size_t(g.ny) * k)
                                              : size_t(s) + size_t(g.nx) * (size_t(p) + size_t(g.ny) * k),
                                     size_t(g.nx) * g.ny * g.nz, 2);
            const float am = (m & 1) ? acc2[m >> 1].y : acc2[m >> 1].x;
            if (CLASS == 0) x[o] = am;
            else x[o] += am;
        }
    }
#endif
}

__global__ void k_atb_matched_zrays_f32(KGeom g, const float* __restrict__ pg, float* __restrict__ x) {
    const size_t nvox = size_t(g.nx) * g.ny * g.nz;
    const size_t id = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (id >= nvox) return;
    const int i = int(id % g.nx), j = int((id / g.nx) % g.ny), k = int(id / (size_t(g.nx) * g.ny));
    const double h = g.h;
    const int kg = k + g.z0;  // global slice
    const double xc = (i - 0.5 * (g.nx - 1)) * h, yc = (j - 0.5 * (g.ny - 1)) * h, zc = (kg - 0.5 * (g.nzg - 1)) * h;
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
                const float fs = float(kg);
                const float fb = fmaf(fs, w.fbd, w.fb0), fc = fmaf(fs, w.fcd, w.fc0);
                const float fib = floorf(fb), fic = floorf(fc);
                const int ib = int(fib), ic = int(fic);
                const float tb = fb - fib, tc = fc - fic;
                float wb, wc;
                if (i == ib) wb = 1.f - tb; else if (i == ib + 1) wb = tb; else continue;
                if (j == ic) wc = 1.f - tc; else if (j == ic + 1) wc = tc; else continue;
                acc = fmaf(wb * wc, __ldg(pg + chk_idx(g, pg_index(g, a, iu, iv), size_t(g.na) * pg_groups(g.nv) * g.nu * 4, 6)), acc);
            }
        }
    }
    x[id] += acc;
}

// ---- voxel-driven A^T b (projector.hpp:204-279) -----------------------------------------
// Warp = one voxel column (i, j), lanes along z (KZ slices per lane).  Views are taken 32 at
// a time: lane L sets up view a0+L for the column in fp64 -- source offset, perspective
// factor t, detector column fu split into (iu, tu) -- exactly the reference's expressions,
// and the warp then walks the 32 views in order with the per-view values broadcast by
// __shfl_sync (1/32 of the warp-uniform fp64 work per lane instead of all of it).  The row
// position fv = t*z/du + cv is evaluated per sample in fp64 (B200 runs FP64 at half the FP32
// rate) and split into (iv, tv) exactly, so positions round like the reference's double
// positions rather than at ulp(nv) of an f32 coordinate; taps, weights and the per-view sum
// are f32 and the views are summed in the reference's order.
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
    const double xd = (i - 0.5 * (g.nx - 1)) * g.h, yd = (j - 0.5 * (g.ny - 1)) * g.h;
    const double cu = 0.5 * (g.nu - 1), cv = 0.5 * (g.nv - 1);
    const double invdu = 1.0 / g.du;
    const float h = float(g.h);
    const bool cone = g.mode == CTK_CONE3D;
    const bool flat = g.nv == 1;
    float zk[KZ], acc[KZ];
    double zq[KZ];  // z / du
#pragma unroll
    for (int m = 0; m < KZ; ++m) {
        const int k = kb + lane + 32 * m;
        const double z = (k + g.z0 - 0.5 * (g.nzg - 1)) * g.h;
        zk[m] = float(z);
        zq[m] = z * invdu;
        acc[m] = 0.f;
    }
    for (int a0 = 0; a0 < g.na; a0 += 32) {
        // ---- lane L: view a0 + L of this column, fp64 ----
        const int av = a0 + lane;
        double tD = 1.0;
        int iuL = 0;
        float tuL = 0.f, arxy = 0.f, rxy2 = 0.f, spar = 0.f;
        bool ok = false;
        if (av < g.na) {
            const double2 tr = g.ctst[av];
            double fu;
            ok = true;
            if (cone) {
                const double sx = g.dso * tr.x, sy = g.dso * tr.y;
                const double rx = xd - sx, ry = yd - sy;
                const double depth = -(rx * tr.x + ry * tr.y);
                if (depth <= 0.0) ok = false;
                tD = (g.dso + g.dod) / depth;
                const double px = sx + tD * rx, py = sy + tD * ry;
                fu = (-px * tr.y + py * tr.x) * invdu + cu;
                arxy = float(fmax(fabs(rx), fabs(ry)));
                rxy2 = float(rx * rx + ry * ry);
            } else {
                fu = (-xd * tr.y + yd * tr.x) * invdu + cu;
                spar = float(g.h / fmax(fabs(tr.x), fabs(tr.y)));
            }
            if (ok && fu > -2.0 && fu < double(g.nu)) {
                dsplit(fu, iuL, tuL);
                if (iuL < -1 || iuL >= g.nu) ok = false;
            } else {
                ok = false;
            }
        }
        unsigned live = __ballot_sync(0xffffffffu, ok);
        while (live) {  // views in ascending order
            const int L = __ffs(live) - 1;
            live &= live - 1;
            const int a = a0 + L;
            const double t = __shfl_sync(0xffffffffu, tD, L);
            const int iu = __shfl_sync(0xffffffffu, iuL, L);
            const float tu = __shfl_sync(0xffffffffu, tuL, L);
            const float vax = __shfl_sync(0xffffffffu, arxy, L), vr2 = __shfl_sync(0xffffffffu, rxy2, L);
            const float vsp = __shfl_sync(0xffffffffu, spar, L);
            const bool u0ok = iu >= 0, u1ok = iu + 1 < g.nu;
            CTK_CHK(g, a < g.na && iu >= -1 && iu < g.nu, 5);
            const float* c0 = pt + size_t(a * g.nu + iu) * g.nv;
            const float* c1 = c0 + g.nv;
#pragma unroll
            for (int m = 0; m < KZ; ++m) {
                const int k = kb + lane + 32 * m;
                if (k >= g.nz) break;
                int iv = 0;
                float tv = 0.f;
                if (!flat)  // clamped far outside the detector so the split stays exact (taps then read nothing)
                    dsplit(fmin(fmax(__fma_rn(cone ? t : 1.0, zq[m], cv), -4.0), g.nv + 4.0), iv, tv);
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
                    const float z = zk[m];
                    scale = h * sqrtf(fmaf(z, z, vr2)) / fmaxf(vax, fabsf(z));
                } else {
                    scale = vsp;
                }
                acc[m] = fmaf(scale, sample, acc[m]);
            }
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

void transpose_proj(Geometry& g, const float* y, cudaStream_t s) {
    g.proj_t.ensure(g.range() * sizeof(float));
    dim3 blk(32, 8), grd((g.nu + 31) / 32, (g.nv + 31) / 32, g.na);
    k_proj_transpose<<<grd, blk, 0, s>>>(g.kgeom(), y, g.proj_t.as<float>());
    after_launch("k_proj_transpose");
}

void group_proj(Geometry& g, const float* y, cudaStream_t s) {
    const int nq = pg_groups(g.nv);
    g.proj_t.ensure(size_t(g.na) * g.nu * nq * 4 * sizeof(float));
    dim3 blk(32, 8), grd((g.nu + 31) / 32, (nq + 7) / 8, g.na);
    k_proj_group4<<<grd, blk, 0, s>>>(g.kgeom(), y, g.proj_t.as<float>());
    after_launch("k_proj_group4");
}

template <int CLASS, int PB>
void launch_plane_pb(Geometry& g, float* x, cudaStream_t s) {
    constexpr int BP_PB = PB, BP_SL = PlaneCfg<PB>::SL;
    const int nh = CLASS ? g.nx : g.ny;
    const int planes = CLASS ? g.ny : g.nx;
    const int ptiles = (nh + BP_PB - 1) / BP_PB;
    const int kbands = (g.nz_local() + BP_KB - 1) / BP_KB;
    constexpr int NL = CTK_BP_PAIR ? PB / 2 : PB;
    const size_t smem = sizeof(float) * (size_t(z_stride<PB>()) * (BP_KB + 2 * BP_ZG) + size_t(NL) * BP_SL + NL + BP_PB +
                                         4 * size_t(pg_groups(g.nv))) +
                        sizeof(int2) * g.na + sizeof(int) * (size_t(g.na) + 1 + BP_PB);
    if (smem > 200 * 1024) fail(CTK_E_UNSUPPORTED, "too many views / detector rows for the plane backprojector");
    // opt in once to the largest size this launcher accepts (occupancy follows the size of
    // each launch, not the opt-in); call_once keeps concurrent handles on other threads safe
    static std::once_flag opted[64];  // function attributes are per device
    int dev = 0;
    CTK_CUDA(cudaGetDevice(&dev));
    std::call_once(opted[dev & 63], [] {
        CTK_CUDA(cudaFuncSetAttribute(k_atb_plane_f32<CLASS, PB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      200 * 1024));
    });
    dim3 grd(unsigned(planes), unsigned(ptiles * kbands));
    k_atb_plane_f32<CLASS, PB><<<grd, BP_PB, smem, s>>>(g.kgeom(), g.proj_t.as<float>(), x, ptiles);
    after_launch("k_atb_plane_f32");
}

template <int CLASS>
void launch_plane(Geometry& g, float* x, cudaStream_t s) {
    const int nh = CLASS ? g.nx : g.ny;
    static const int forced = [] {
        const char* e = std::getenv("CTK_BP_TILE");  // A/B timing: 128 or 256
        return e ? std::atoi(e) : 0;
    }();
    const int pb = forced == 128 || forced == 256 ? forced : (nh <= 768 ? 128 : 256);
    if (pb == 128) launch_plane_pb<CLASS, 128>(g, x, s);
    else launch_plane_pb<CLASS, 256>(g, x, s);
}

template <int KZ>
void launch_voxel(Geometry& g, float* x, cudaStream_t s) {
    const int kblocks = (g.nz_local() + 32 * KZ - 1) / (32 * KZ);
    const long warps = long(g.nx) * g.ny * kblocks;
    dim3 blk(32, 4);
    const unsigned grd = unsigned((warps + 3) / 4);
    k_atb_voxel_f32<KZ><<<grd, blk, 0, s>>>(g.kgeom(), g.proj_t.as<float>(), x, kblocks);
    after_launch("k_atb_voxel_f32");
}

}  // namespace

void atb_matched_f32(Geometry& g, const float* y, float* x, cudaStream_t s) {
    group_proj(g, y, s);
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
    transpose_proj(g, y, s);
    CTK_CUDA(cudaEventRecord(g.ev0, s));
    switch (pick_kz(g.nz_local())) {
        case 1: launch_voxel<1>(g, x, s); break;
        case 2: launch_voxel<2>(g, x, s); break;
        case 4: launch_voxel<4>(g, x, s); break;
        case 8: launch_voxel<8>(g, x, s); break;
        default: launch_voxel<16>(g, x, s); break;
    }
    CTK_CUDA(cudaEventRecord(g.ev1, s));
}

}  // namespace ctkb
