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
    const float* fr = y + size_t(a) * g.nu * g.nw;  // rows held: [w0, w0 + nw), local index iv
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int iu = u0 + threadIdx.x, iv = v0 + r;
        tile[r][threadIdx.x] = (iu < g.nu && iv < g.nw) ? __ldg(fr + size_t(iv) * g.nu + iu) : 0.f;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int iu = u0 + r, iv = v0 + threadIdx.x;
        if (iu < g.nu && iv < g.nw) {
            pt[(size_t(a) * g.nu + iu) * g.nw + iv] = tile[threadIdx.x][r];
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
    return ((size_t(a) * pg_groups(g.nw) + (iv >> 2)) * g.nu + iu) * 4 + (iv & 3);  // iv local (held rows)
}

__global__ void k_proj_group4(KGeom g, const float* __restrict__ y, float* __restrict__ pg) {
    // block: 32 columns x 8 row groups; thread (u, q) writes one float4
    const int a = blockIdx.z;
    const int iu = blockIdx.x * 32 + threadIdx.x, q = blockIdx.y * 8 + threadIdx.y;
    const int nq = pg_groups(g.nw);  // groups of the held rows [w0, w0 + nw)
    if (iu >= g.nu || q >= nq) return;
    const int c = a * g.nu + iu;
    const double2 cs = g.colstep[c];
    const float* fr = y + size_t(a) * g.nu * g.nw;
    float r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int iv = 4 * q + j;  // local row
        r[j] = iv < g.nw ? __ldg(fr + size_t(iv) * g.nu + iu) * ray_step(g, cs, row_coord(g, g.w0 + iv)) : 0.f;
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
//           the slots registered in its row: a per-row bit mask over the batch's slots,
//           walked with __ffs in slot order -> deterministic, the (view, column) order.
//           (Round 1 kept sorted per-row lists of up to 11 entries with an overflow scan;
//           the masks take 1 KB less shared memory, one 16-byte load per row, no sort.)
// Z[k][e] has row stride BP_PB: phase-1 lanes (consecutive e) hit distinct banks whatever
// their k, phase-2 lanes (consecutive rows -> consecutive e) likewise.
// Tile size PB (rows = threads per CTA) is a template parameter with its own occupancy
// (round 1, matched A^T b f32): PB = 128, 6 CTAs/SM: 512^3/360 66.9 ms; PB = 256, 3 CTAs/SM:
// 512^3/360 72.8 ms, 1024^3/1600 2518 ms (PB = 128: 3034 ms -- per-CTA setup over 1600
// views, twice the tiles); with the registration masks PB = 256 pays only beyond 768 rows
// per plane AND about 1000 views (launch_plane).
// 128-row tiles: 6 blocks/SM at 80 registers (7 / 8 blocks: 72 / 64 registers with spills,
// 73.0 / 81.2 ms vs 71.1 at C3)
#ifndef CTK_BP_MINB128
#define CTK_BP_MINB128 6
#endif
template <int PB>
struct PlaneCfg;
template <>
struct PlaneCfg<128> {
    static constexpr int MINB = CTK_BP_MINB128;
};
template <>
struct PlaneCfg<256> {
    static constexpr int MINB = 3;
};
#ifndef CTK_BP_KB
#define CTK_BP_KB 32
#endif
constexpr int BP_KB = CTK_BP_KB;
constexpr int BP_ZG = 2;
// Z row stride (a multiple of the 32 banks: phase-1 lanes, consecutive slots, never conflict)
template <int PB>
__host__ __device__ constexpr int z_stride() { return PB; }
__device__ __forceinline__ int z_col(int e) { return e; }
  // guard rows of Z on each side: out-of-band entries land there, unread

// SID = 1: the transpose of the f32 Siddon forward (f32_common.cuh model) in the same
// structure: phase 1 fills two Z columns per slot (the column's two in-plane cells at the
// plane), each registered in its row with weight 1 (L is in pg).
template <int CLASS, int PB, int SID = 0, int WIN = 0>
__global__ void __launch_bounds__(PB, PlaneCfg<PB>::MINB)
k_atb_plane_f32(KGeom g, const float* __restrict__ pg, float* __restrict__ x, int ptiles, int nvc) {
    // WIN: the band-sharded range's row window (W0, NW); else the whole detector, with
    // the window folded to constants so the common case keeps its register allocation
    const int W0 = WIN ? g.w0 : 0, NW = WIN ? g.nw : g.nv;
    constexpr int BP_PB = PB;
    constexpr int MW = PB / 32;  // registration mask words per row
    extern __shared__ __align__(16) float sm[];
    constexpr int ZS = z_stride<PB>();                          // row stride of Z
    float* Z = sm + BP_ZG * ZS;                                 // [-BP_ZG, BP_KB+BP_ZG) x [ZS]
    float* Z2 = Z + (BP_KB + 2 * BP_ZG) * ZS;                   // Siddon: the second in-plane cell
    // registration: bit e of row p's mask <=> slot e touches row p (its in-plane stencil rows
    // are eih[e] and eih[e] + 1, with weights 1 - eth[e] and eth[e]; Siddon: its cells)
    unsigned* rmask = reinterpret_cast<unsigned*>(Z + (BP_KB + BP_ZG + (SID ? BP_KB + 2 * BP_ZG : 0)) * ZS);  // [PB][MW]
    int* eih = reinterpret_cast<int*>(rmask + BP_PB * MW);     // [BP_PB]
    float* eth = reinterpret_cast<float*>(eih + BP_PB);         // [BP_PB]
    static_assert(MW % 4 == 0 && BP_PB % 4 == 0, "keeps the masks and vrtab 16-byte aligned");
    const int nv4 = 4 * pg_groups(NW);  // held rows, local index (band-sharded range)
    float* vrtab = eth + BP_PB;                                 // [nv4] iv - (nv-1)/2, 16-byte aligned
    float* ivrtab = vrtab + (SID ? nv4 : 0);                    // Siddon: [nv4] 1/|iv - (nv-1)/2|
    int2* urange = reinterpret_cast<int2*>(vrtab + (SID ? 2 : 1) * nv4);  // [na]
    int* pref = reinterpret_cast<int*>(urange + g.na);          // [na + 1] candidate prefix sums

    const int t = threadIdx.x;
    // plane index fastest: a wave of resident CTAs shares one (row tile, z band), so per
    // view it reads only that band's detector rows -> the projections stay L2-resident
    const int s = blockIdx.x;
    // view chunks (small problems): CTA chunk vc sums the views [a_lo, a_hi) into its own
    // partial volume x + vc * N (k_sum_parts adds the chunks in order afterwards)
    const int vch = blockIdx.y % nvc, ptk = blockIdx.y / nvc;
    const int a_lo = int((long(vch) * g.na) / nvc), a_hi = int((long(vch + 1) * g.na) / nvc);
    x += size_t(vch) * size_t(g.nx) * g.ny * g.nz;
    const int ptile = ptk % ptiles, kband = ptk / ptiles;
    const int p0 = ptile * BP_PB, k0 = kband * BP_KB;
    const int nh = CLASS ? g.nx : g.ny;
    const int p = p0 + t;
    for (int q = t; q < nv4; q += BP_PB) {
        vrtab[q] = row_vr(g, W0 + q);
        if (SID) ivrtab[q] = __frcp_rn(fabsf(row_vr(g, W0 + q)));
    }
    const int sc = slice_centre(s);  // anchored positions (f32_common.cuh): block centre of plane s
    const float kf = float(s - sc);
    const float czf = 0.5f * float(g.nzg - 1);  // global z centre; this handle's slices start at z0
    const int kg0 = k0 + g.z0;                   // global index of the band's first slice
    const float cvf = 0.5f * float(g.nv - 1);
    const float invdu = float(1.0 / g.du);
    const float fs = float(s);
    const double h = g.h;
    const int nq = pg_groups(NW);  // row groups of the grouped projection layout
    // world coordinates of the plane and of the tile's row segment ends
    const double plane_c = (s - 0.5 * ((CLASS ? g.ny : g.nx) - 1)) * h;
    const double r_lo = (p0 - (SID ? 2.5 : 1.5) - 0.5 * (nh - 1)) * h,
                 r_hi = (p0 + BP_PB + (SID ? 1.5 : 0.5) - 0.5 * (nh - 1)) * h;

    // BP_KB accumulators as packed pairs: phase 2 adds wh * Z with FFMA2 (per element the
    // scalar fma)
    float2 acc2[BP_KB / 2];
#pragma unroll
    for (int m = 0; m < BP_KB / 2; ++m) acc2[m] = make_float2(0.f, 0.f);
    auto add_sid = [&](const float* Zw, int e) {  // Siddon: weight 1
        const int ze = z_col(e);
#pragma unroll
        for (int m = 0; m < BP_KB / 2; ++m)
            acc2[m] = __fadd2_rn(make_float2(Zw[(2 * m) * ZS + ze], Zw[(2 * m + 1) * ZS + ze]), acc2[m]);
    };
    // a Siddon slot was processed (and registered) iff its cells meet this tile
    auto jlo_ok = [&](int ja, int jb) {
        const int jlo = min(ja, jb), jhi = max(ja, jb);
        return jhi >= p0 && jlo <= p0 + BP_PB - 1 && jhi >= 0 && jlo < nh;
    };
    auto add_entry = [&](float wh, int e) {
        const float2 w2 = make_float2(wh, wh);
        const int ze = z_col(e);
#pragma unroll
        for (int m = 0; m < BP_KB / 2; ++m)
            acc2[m] = __ffma2_rn(w2, make_float2(Z[(2 * m) * ZS + ze], Z[(2 * m + 1) * ZS + ze]), acc2[m]);
    };

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
        if (a < a_lo || a >= a_hi) i1 = i0 - 1;  // another view chunk's
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
#pragma unroll
            for (int w = 0; w < MW; w += 4) *reinterpret_cast<uint4*>(rmask + t * MW + w) = make_uint4(0u, 0u, 0u, 0u);
            int a = -1, iu = 0;
            const int gidx = b0 + t;
            if (gidx < total) {  // the view of this slot: pref[a] <= gidx < pref[a + 1]
                while (pref[a_run + 1] <= gidx) ++a_run;  // monotone over batches: ~1 step
                a = a_run;
                iu = urange[a].x + (gidx - pref[a]);
            }
            __syncthreads();
            if (a >= 0) {
                const int c = a * g.nu + iu;
                if (g.colaxis[c] == CLASS) {
                if constexpr (SID) {
                    // ---- Siddon phase 1 (f32_common.cuh model): the column's cell ja at the
                    // plane's t = 0 boundary and jb = ja +- 1 when the chord crosses a y boundary
                    // (cy < 1); every row adds its four chord weights times (L y) to Z (cell ja)
                    // and Z2 (cell jb) at its z cells ka, kb -- rolled over (kl, kl + 1),
                    // kl = min(ka, kb) non-decreasing in iv
                    const float4 cd = g.col[c];
                    const double4 c64 = g.col64[c];
                    int jA, ja;
                    float tA, fya;
                    double G;
                    sid_anchor(c64, sc, jA, tA, G);
                    split(fmaf(kf - 0.5f, cd.y, tA), ja, fya);
                    ja += jA;
                    const bool incy = cd.y >= 0.f;
                    const float cy = sid_cross(fya, sid_coef(incy, __frcp_rn(fabsf(cd.y))));
                    const int jb = cy < 1.f ? (incy ? ja + 1 : ja - 1) : ja;
                    if (jlo_ok(ja, jb)) {
                        const float gs = fmaf(fs, cd.w, cd.z);
                        int v0 = 0, v1 = g.nv - 1;
                        if (gs > 0.f) {
                            const float rg = invdu / gs;
                            // a row reaches the band iff its centre-plane fz lies in
                            // [kg0 - 2, kg0 + KB) (cells kl, kl+1 at the slab boundaries, which are
                            // within half a slice of the centre plane); one row of margin
                            v0 = max(v0, int(floorf(fmaf(float(kg0) - 2.f - czf, rg, cvf))) - 1);
                            v1 = min(v1, int(ceilf(fmaf(float(kg0 + BP_KB) - czf, rg, cvf))) + 1);
                        }
                        if (g.has_zrays) {  // z-dominant rows: the exact gather (siddon.cu, zonly)
                            const double dA = g.colstep[c].y;
                            const double cv = 0.5 * (g.nv - 1), r = dA / g.du;
                            int lo = max(v0, int(ceil(cv - r)) - 1), hi = min(v1, int(floor(cv + r)) + 1);
                            while (lo <= hi && fabs(row_coord(g, lo)) > dA) ++lo;
                            while (hi >= lo && fabs(row_coord(g, hi)) > dA) --hi;
                            v0 = lo;
                            v1 = hi;
                        }
                        if constexpr (WIN) {  // held rows, local index
                            v0 = max(v0, W0) - W0;
                            v1 = min(v1, W0 + NW - 1) - W0;
                        }
                        const float4* pc4 = reinterpret_cast<const float4*>(pg) + size_t(a) * nq * g.nu + iu;
                        const size_t qs = size_t(g.nu);
                        float* zc = Z + z_col(t);
                        float* zc2 = Z2 + z_col(t);
                        float Whi, Wr;
                        z_split(g, G, Whi, Wr);
                        const float Wd = z_cross(g, c64), aWd = __frcp_rn(fabsf(Wd)), fcs = sid_fc(g);
                        const float Wa = fmaf(kf - 0.5f, Wd, Wr);
                        const int koff = sid_izc(g) - kSplitBias - kg0;
                        // one row: its z cells and four weights, the forward's expressions
                        // (1/|vr| from the shared table = __frcp_rn(|vr|))
                        auto row_w = [&](int iv, int& kl, float& a0, float& a1, float& b0, float& b1) {
                            const float vr = vrtab[iv];
                            const float S = fmaf(vr, Whi, fcs);
                            const float tta = split_t(fmaf(vr, Wa, S));
                            const float fza = fmaf(vr, Wa, fmaf(__fsub_rn(tta, kSplitM), -1.f, S));
                            const int ka = __float_as_int(tta) + koff;
                            const bool incz = vr * Wd >= 0.f;
                            const float cz = sid_cross(fza, sid_coef(incz, ivrtab[iv] * aWd));
                            const float m = fminf(cy, cz), M = fmaxf(cy, cz);
                            const float wff = m, wfs = cy - m, wsf = cz - m, wss = 1.f - M;
                            const bool lowfirst = incz || !(cz < 1.f);  // ka <= kb
                            kl = lowfirst ? ka : ka - 1;
                            a0 = lowfirst ? wff : wfs;
                            a1 = lowfirst ? wfs : wff;
                            b0 = lowfirst ? wsf : wss;
                            b1 = lowfirst ? wss : wsf;
                        };
                        auto zero_rows = [&](int lo, int hi) {
                            for (int m = max(lo, 0); m < min(hi, BP_KB); ++m) zc[m * ZS] = zc2[m * ZS] = 0.f;
                        };
                        if (gs > 0.f && v0 <= v1) {
                            // the rolling march of the Joseph pass over whole 4-row groups (rows
                            // outside [v0, v1] masked to zero), two Z columns
                            const float rg = invdu / gs;
                            const int q0 = v0 >> 2, q1 = v1 >> 2;
                            CTK_CHK(g, q0 >= 0 && q1 < nq, 1);
                            int kl0;
                            float u0, u1, u2, u3;
                            row_w(4 * q0, kl0, u0, u1, u2, u3);
                            zero_rows(0, rg >= 0.75f ? kl0 : BP_KB);
                            int cur = -(1 << 20);
                            float A = 0.f, B = 0.f, C = 0.f, D = 0.f;
                            auto rowstep = [&](int iv, float yv) {
                                int kk;
                                float a0, a1, b0, b1;
                                row_w(iv, kk, a0, a1, b0, b1);
                                const int adv = kk - cur;
                                float ak = adv == 1 ? B : 0.f, ck = adv == 1 ? D : 0.f;
                                ak = adv == 0 ? A : ak;
                                ck = adv == 0 ? C : ck;
                                const float bk = adv == 0 ? B : 0.f, dk = adv == 0 ? D : 0.f;
                                A = fmaf(a0, yv, ak);
                                B = fmaf(a1, yv, bk);
                                C = fmaf(b0, yv, ck);
                                D = fmaf(b1, yv, dk);
                                cur = kk;
                                const unsigned r = min(unsigned(kk + BP_ZG), unsigned(BP_KB + 2 * BP_ZG - 2));
                                float* zp = zc - BP_ZG * ZS + r * ZS;
                                float* zp2 = zc2 - BP_ZG * ZS + r * ZS;
                                zp[0] = A;
                                zp[ZS] = B;
                                zp2[0] = C;
                                zp2[ZS] = D;
                            };
                            auto group = [&](int q, float4 y4, bool mask) {
                                const int b = 4 * q;
                                if (mask) {
                                    y4.x = (b >= v0 && b <= v1) ? y4.x : 0.f;
                                    y4.y = (b + 1 >= v0 && b + 1 <= v1) ? y4.y : 0.f;
                                    y4.z = (b + 2 >= v0 && b + 2 <= v1) ? y4.z : 0.f;
                                    y4.w = (b + 3 >= v0 && b + 3 <= v1) ? y4.w : 0.f;
                                }
                                rowstep(b, y4.x);
                                rowstep(b + 1, y4.y);
                                rowstep(b + 2, y4.z);
                                rowstep(b + 3, y4.w);
                            };
                            group(q0, __ldg(pc4 + q0 * qs), true);
                            for (int q = q0 + 1; q < q1; ++q) group(q, __ldg(pc4 + q * qs), false);
                            if (q1 > q0) group(q1, __ldg(pc4 + q1 * qs), true);
                            zero_rows(cur + 2, BP_KB);
                        } else {
                            zero_rows(0, BP_KB);
                            for (int iv = v0; iv <= v1; ++iv) {
                                const float yv = __ldg(reinterpret_cast<const float*>(pc4 + (iv >> 2) * qs) + (iv & 3));
                                int kk;
                                float a0, a1, b0, b1;
                                row_w(iv, kk, a0, a1, b0, b1);
                                if (unsigned(kk) < unsigned(BP_KB)) {
                                    zc[kk * ZS] = fmaf(a0, yv, zc[kk * ZS]);
                                    zc2[kk * ZS] = fmaf(b0, yv, zc2[kk * ZS]);
                                }
                                if (unsigned(kk + 1) < unsigned(BP_KB)) {
                                    zc[(kk + 1) * ZS] = fmaf(a1, yv, zc[(kk + 1) * ZS]);
                                    zc2[(kk + 1) * ZS] = fmaf(b1, yv, zc2[(kk + 1) * ZS]);
                                }
                            }
                        }
                        // register: row ja reads Z, row jb != ja reads Z2
                        eih[t] = ja;
                        if (ja >= p0 && ja <= p0 + BP_PB - 1 && ja >= 0 && ja < nh)
                            atomicOr(&rmask[(ja - p0) * MW + (t >> 5)], 1u << (t & 31));
                        if (jb != ja && jb >= p0 && jb <= p0 + BP_PB - 1 && jb >= 0 && jb < nh)
                            atomicOr(&rmask[(jb - p0) * MW + (t >> 5)], 1u << (t & 31));
                    }
                } else {
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
                        if constexpr (WIN) {  // the held rows, local index from here on
                            v0 = max(v0, W0) - W0;
                            v1 = min(v1, W0 + NW - 1) - W0;
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
                        eih[t] = ih;
                        if (ih >= p0) atomicOr(&rmask[(ih - p0) * MW + (t >> 5)], 1u << (t & 31));
                        if (ih + 1 <= p0 + BP_PB - 1 && th != 0.f)
                            atomicOr(&rmask[(ih + 1 - p0) * MW + (t >> 5)], 1u << (t & 31));
                    }
                }
                }
            }
            __syncthreads();
            // ---- phase 2: row p gathers its registered slots in slot order, i.e. in (view,
            // column) order: deterministic, and the order of the reference's scatter ----
            if (p < nh) {
                // 64-bit words (half the word steps of 32-bit ones: C3 72.5 -> 70.9 ms)
#pragma unroll
                for (int w4 = 0; w4 < MW; w4 += 4) {
                    const ulonglong2 m2 = *reinterpret_cast<const ulonglong2*>(rmask + t * MW + w4);
                    const unsigned long long mw[2] = {m2.x, m2.y};
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        unsigned long long bits = mw[j];
                        while (bits) {
                            const int e = (w4 + 2 * j) * 32 + __ffsll(bits) - 1;
                            bits &= bits - 1;
                            if constexpr (SID) {
                                add_sid(eih[e] == p ? Z : Z2, e);
                            } else {
                                const float th = eth[e];
                                add_entry(eih[e] == p ? 1.f - th : th, e);
                            }
                        }
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
            const size_t o = chk_idx(g, CLASS ? size_t(p) + size_t(g.nx) * (size_t(s) + size_t(g.ny) * k)
                                              : size_t(s) + size_t(g.nx) * (size_t(p) + size_t(g.ny) * k),
                                     size_t(g.nx) * g.ny * g.nz, 2);
            const float am = (m & 1) ? acc2[m >> 1].y : acc2[m >> 1].x;
            if (CLASS == 0) x[o] = am;
            else x[o] += am;
        }
    }
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
        iv0 = max(iv0, g.w0);  // the held rows (band-sharded range)
        iv1 = min(iv1, g.w0 + g.nw - 1);
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
                acc = fmaf(wb * wc, __ldg(pg + chk_idx(g, pg_index(g, a, iu, iv - g.w0), size_t(g.na) * pg_groups(g.nw) * g.nu * 4, 6)), acc);
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
            const float* c0 = pt + (ptrdiff_t(a * g.nu + iu) * g.nw - g.w0);  // by global row; rows held [w0, w0+nw)
            const float* c1 = c0 + g.nw;
#pragma unroll
            for (int m = 0; m < KZ; ++m) {
                const int k = kb + lane + 32 * m;
                if (k >= g.nz) break;
                int iv = 0;
                float tv = 0.f;
                if (!flat)  // clamped far outside the detector so the split stays exact (taps then read nothing)
                    dsplit(fmin(fmax(__fma_rn(cone ? t : 1.0, zq[m], cv), -4.0), g.nv + 4.0), iv, tv);
                const bool v0ok = iv >= g.w0 && iv < g.w0 + g.nw, v1ok = iv + 1 >= g.w0 && iv + 1 < g.w0 + g.nw;
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
    dim3 blk(32, 8), grd((g.nu + 31) / 32, (g.rows_local() + 31) / 32, g.na);
    k_proj_transpose<<<grd, blk, 0, s>>>(g.kgeom(), y, g.proj_t.as<float>());
    after_launch("k_proj_transpose");
}

void group_proj(Geometry& g, const float* y, cudaStream_t s) {
    const int nq = pg_groups(g.rows_local());
    g.proj_t.ensure(size_t(g.na) * g.nu * nq * 4 * sizeof(float));
    dim3 blk(32, 8), grd((g.nu + 31) / 32, (nq + 7) / 8, g.na);
    k_proj_group4<<<grd, blk, 0, s>>>(g.kgeom(), y, g.proj_t.as<float>());
    after_launch("k_proj_group4");
}

template <int CLASS, int PB, int SID, int WIN>
void launch_plane_pb(Geometry& g, float* x, cudaStream_t s, int nvc) {
    constexpr int BP_PB = PB;
    const int nh = CLASS ? g.nx : g.ny;
    const int planes = CLASS ? g.ny : g.nx;
    const int ptiles = (nh + BP_PB - 1) / BP_PB;
    const int kbands = (g.nz_local() + BP_KB - 1) / BP_KB;
    const size_t smem = sizeof(float) * (size_t(z_stride<PB>()) * (BP_KB + 2 * BP_ZG) * (SID ? 2 : 1) +
                                         size_t(BP_PB) * (BP_PB / 32) + 2 * BP_PB +
                                         4 * size_t(pg_groups(g.rows_local())) * (SID ? 2 : 1)) +
                        sizeof(int2) * g.na + sizeof(int) * (size_t(g.na) + 1);
    if (smem > 200 * 1024) fail(CTK_E_UNSUPPORTED, "too many views / detector rows for the plane backprojector");
    // opt in once to the largest size this launcher accepts (occupancy follows the size of
    // each launch, not the opt-in); call_once keeps concurrent handles on other threads safe
    static std::once_flag opted[64];  // function attributes are per device
    int dev = 0;
    CTK_CUDA(cudaGetDevice(&dev));
    std::call_once(opted[dev & 63], [] {
        CTK_CUDA(cudaFuncSetAttribute(k_atb_plane_f32<CLASS, PB, SID, WIN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      200 * 1024));
    });
    dim3 grd(unsigned(planes), unsigned(ptiles * kbands * nvc));
    k_atb_plane_f32<CLASS, PB, SID, WIN><<<grd, BP_PB, smem, s>>>(g.kgeom(), g.proj_t.as<float>(), x, ptiles, nvc);
    after_launch(SID ? "k_atb_plane_f32_siddon" : "k_atb_plane_f32");
}

template <int CLASS>
void launch_plane(Geometry& g, float* x, cudaStream_t s, int nvc) {
    const int nh = CLASS ? g.nx : g.ny;
    static const int forced = [] {
        const char* e = std::getenv("CTK_BP_TILE");  // A/B timing: 128 or 256
        return e ? std::atoi(e) : 0;
    }();
    // 256-row tiles halve the CTAs, i.e. the per-CTA setup over all views: measured with the
    // registration masks at 1024^3, 400 views 680 vs 628 ms (128 wins), 1600 views 2778 vs
    // 2859 ms (256 wins); 512^3/720: 128 wins (142 vs 154 ms)
    const int pb = forced == 128 || forced == 256 ? forced : (nh > 768 && g.na >= 1000 ? 256 : 128);
    const bool sid = g.projector == CTK_PROJ_SIDDON;  // (Siddon has no band-sharded range)
    if (pb == 128) {
        if (sid) launch_plane_pb<CLASS, 128, 1, 0>(g, x, s, nvc);
        else if (g.band) launch_plane_pb<CLASS, 128, 0, 1>(g, x, s, nvc);
        else launch_plane_pb<CLASS, 128, 0, 0>(g, x, s, nvc);
    } else {
        if (sid) launch_plane_pb<CLASS, 256, 1, 0>(g, x, s, nvc);
        else if (g.band) launch_plane_pb<CLASS, 256, 0, 1>(g, x, s, nvc);
        else launch_plane_pb<CLASS, 256, 0, 0>(g, x, s, nvc);
    }
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

// View chunks of the plane A^T b: a small problem launches fewer (plane, tile, band) CTAs
// than one wave of the GPU (C1: 128 against 148 SMs x 6) and each loops over every view;
// splitting the views into nvc chunks multiplies the CTAs, each chunk summing into its own
// partial volume, added in chunk order afterwards (deterministic)
int view_chunks(const Geometry& g) {
    static const int forced = [] {
        const char* e = std::getenv("CTK_BP_VCHUNKS");  // A/B timing
        return e ? std::max(1, std::atoi(e)) : 0;
    }();
    if (forced) return std::min(forced, std::max(1, g.na));
    const int nh = std::max(g.nx, g.ny), pb = nh <= 768 ? 128 : 256;
    const long ctas = long(std::max(g.nx, g.ny)) * ((nh + pb - 1) / pb) * ((g.nz_local() + BP_KB - 1) / BP_KB);
    const long wave = 148L * (pb == 128 ? 6 : 3);
    // measured at C1 (64^3/100, 128 CTAs per pass): 1 / 4 / 8 chunks 0.279 / 0.129 / 0.138 ms; at
    // 128^3 (512 CTAs) 2 chunks lose 2 %: chunk only while a pass fills less than half a wave
    return int(std::max(1L, std::min(std::min(4L, long(g.na)), wave / ctas)));
}

__global__ void k_sum_parts(size_t n, int nparts, const float* __restrict__ parts, float* __restrict__ x) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        float acc = parts[i];
        for (int q = 1; q < nparts; ++q) acc += parts[size_t(q) * n + i];
        x[i] = acc;
    }
}

void atb_matched_f32(Geometry& g, const float* y, float* x, cudaStream_t s) {
    group_proj(g, y, s);
    const int nvc = view_chunks(g);
    float* xt = x;
    if (nvc > 1) {
        g.bp_parts_buf.ensure(size_t(nvc) * g.domain() * sizeof(float));
        xt = g.bp_parts_buf.as<float>();
    }
    CTK_CUDA(cudaEventRecord(g.ev0, s));
    launch_plane<0>(g, xt, s, nvc);
    launch_plane<1>(g, xt, s, nvc);
    if (nvc > 1) {
        const size_t n = g.domain();
        k_sum_parts<<<unsigned(std::min<size_t>((n + 255) / 256, 148 * 16)), 256, 0, s>>>(n, nvc, xt, x);
        after_launch("k_sum_parts");
    }
    CTK_CUDA(cudaEventRecord(g.ev1, s));
    if (g.has_zrays && g.projector == CTK_PROJ_SIDDON) {
        siddon_atb_zrays_f32(g, y, x, s);  // exact gather of the z-dominant rays, accumulated
    } else if (g.has_zrays) {
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
