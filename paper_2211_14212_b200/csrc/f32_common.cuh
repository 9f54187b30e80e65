// Shared device helpers of the f32 performance kernels (fwd_f32.cu, bp_f32.cu).
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
#pragma once
#include <cfloat>

#include "ctk_internal.h"
#include "reduce.cuh"

namespace ctkb {
namespace {

// Bounds checks of the checked build (ops.cpp check_bounds): record bit `bit` when idx is
// outside [0, n) and return a safe index (0) so the access itself stays in bounds.
#ifdef CTK_CHECKED
template <class I>
__device__ __forceinline__ I chk_idx(const KGeom& g, I idx, I n, int bit) {
    if (idx < I(0) || idx >= n) {
        atomicOr(g.chk, 1u << bit);
        return I(0);
    }
    return idx;
}
#define CTK_CHK(g, cond, bit) \
    do {                       \
        if (!(cond)) atomicOr((g).chk, 1u << (bit)); \
    } while (0)
#else
template <class I>
__device__ __forceinline__ I chk_idx(const KGeom&, I idx, I, int) { return idx; }
#define CTK_CHK(g, cond, bit) \
    do {                       \
    } while (0)
#endif

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
    const int n3[3] = {g.nx, g.ny, g.nzg};  // global geometry; a slab is applied in the march
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

// z-rays only (axis 2): slices are global z, restricted to the handle's slab
__device__ float march_generic(const KGeom& g, const WalkF& w, const float* __restrict__ vol) {
    int s0 = g.z0, s1 = g.z0 + g.nz - 1;
    clip_affine(w.fb0, w.fbd, -1.0, w.nb, s0, s1);
    clip_affine(w.fc0, w.fcd, -1.0, w.nc, s0, s1);
    float acc = 0.f;
    for (int s = s0; s <= s1; ++s) {
        const float fb = fmaf(float(s), w.fbd, w.fb0);
        const float fc = fmaf(float(s), w.fcd, w.fc0);
        const float fib = floorf(fb), fic = floorf(fc);
        const int ib = int(fib), ic = int(fic);
        const float tb = fb - fib, tc = fc - fic;
        const float* p = vol + size_t(s - g.z0) * w.sa;
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

// floor without the conversion pipe: t = f + 1.5*2^23 rounded toward -inf (one FADD.RM) is
// exactly 1.5*2^23 + floor(f) for |f| < 2^22, so its bit pattern minus that of 1.5*2^23 is
// floor(f) and f - (t - 1.5*2^23) the exact fraction in [0, 1).
constexpr float kSplitM = 12582912.0f;
constexpr int kSplitBias = 0x4B400000;  // __float_as_int(kSplitM)
__device__ __forceinline__ float split_t(float f) { return __fadd_rd(f, kSplitM); }
__device__ __forceinline__ float split_frac(float f, float t) { return __fsub_rn(f, __fsub_rn(t, kSplitM)); }
__device__ __forceinline__ void split(float f, int& i, float& frac) {
    const float t = split_t(f);
    i = __float_as_int(t) - kSplitBias;
    frac = split_frac(f, t);
}


// ---- anchored f32 positions (both the forward and the matched transpose) ---------------
// The reference evaluates the sample positions in fp64 even for T = float
// (projector.hpp:97-103): fb = fb0 + s*fb_d, floor, fraction.  A plain f32 evaluation of
// fh(s) = fh0 + s*fhd or fz = vd*G(s) + cz rounds at the magnitude of the coordinate (up to
// n), i.e. ~ulp(512) = 6e-5 voxel at 512^3, which random-signed data expose as ~2e-5
// relative error.  Here positions round at the magnitude of a small offset instead:
//  * in-plane: slices are grouped in blocks of kSB anchored at the block centre sc
//      fh(s) = ihA + fmaf(k, fhd, thA),  k = s - sc in [-kSB/2, kSB/2),
//    with ihA + thA = fh0 + sc*fhd split exactly in fp64;
//  * z: fz(s, iv) = cz + vr*W(s) with vr = iv - (nv-1)/2 and W(s) = du*G(s) (dz per row).
//    W(sc) is split into Whi (12 significant bits) + Wr, so that S = fmaf(vr, Whi, fc) is
//    EXACT in f32 (fc = cz - floor(cz) in {0, 1/2}), and the small rest
//    vr*Wlo, Wlo = fmaf(k, Wd, Wr) (Wd = du*gd), is added to S's fraction:
//      T = fmaf(vr, Wlo, S)          (rounded; only its floor is used)
//      iz = floor(cz) + floor(T),  tz = fmaf(vr, Wlo, S - floor(T))   (S - floor(T) exact)
//    tz can leave [0, 1) by a rounding (1e-7) where T sits on a voxel boundary; the
//    bilinear weights then extrapolate by that amount, a continuous, negligible change.
// The forward (lane = row, loop over s; S per block) and the transpose (thread = column,
// loop over rows at a fixed plane s) evaluate these same expressions with the same
// operands, so positions and weights stay bit-identical between A and A^T.  fp64 parts use
// explicit intrinsics (no contraction differences between the two kernels).
#ifndef CTK_APOS_SB
#define CTK_APOS_SB 32
#endif
constexpr int kSB = CTK_APOS_SB;
static_assert((kSB & (kSB - 1)) == 0, "slice blocks are a power of two");

// floor / exact fraction of an fp64 value (|x| < 2^31): x + 1.5*2^52 rounded down carries
// floor(x) in its low word; the fraction is exact in fp64 and rounded once to f32
__device__ __forceinline__ void dsplit(double x, int& i, float& frac) {
    constexpr double kM52 = 6755399441055744.0;  // 1.5 * 2^52
    const double t = __dadd_rd(x, kM52);
    i = __double2loint(t);
    frac = __double2float_rn(__dsub_rn(x, __dsub_rn(t, kM52)));
}
__device__ __forceinline__ int slice_centre(int s) { return (s & ~(kSB - 1)) + kSB / 2; }
// fh anchor and G(sc) of a column at the block centre sc
__device__ __forceinline__ void slice_anchor(const double4& c, int sc, int& ihA, float& thA, double& G) {
    dsplit(__fma_rn(double(sc), c.y, c.x), ihA, thA);
    G = __fma_rn(double(sc), c.w, c.z);
}
// W = du*G split into Whi (12 significant bits: vr*Whi is exact for |vr| < 2^12) + Wr
__device__ __forceinline__ void z_split(const KGeom& g, double G, float& Whi, float& Wr) {
    const double W = __dmul_rn(g.du, G);
    Whi = __int_as_float(__float_as_int(__double2float_rn(W)) & int(0xFFFFF000u));
    Wr = __double2float_rn(__dsub_rn(W, double(Whi)));
}
// Wd = du*gd: the change of W per slice
__device__ __forceinline__ float z_cross(const KGeom& g, const double4& c) { return __double2float_rn(__dmul_rn(g.du, c.w)); }
// row offset from the detector centre, exact in f32 (half-integers below 2^22)
__device__ __forceinline__ float row_vr(const KGeom& g, int iv) { return float(iv) - 0.5f * float(g.nv - 1); }
// cz = (nzg-1)/2 = izc + fc
__device__ __forceinline__ int cz_int(const KGeom& g) { return (g.nzg - 1) >> 1; }
__device__ __forceinline__ float cz_frac(const KGeom& g) { return ((g.nzg - 1) & 1) ? 0.5f : 0.f; }

// ---- f32 Siddon model (fwd_f32.cu SID = 1, bp_f32.cu SID = 1) ---------------------------
// Siddon's weight of (ray, voxel) is the ray's length inside the voxel box.  Split the ray by
// the slabs of its dominant axis A: slab s spans the boundaries s - 1/2 and s + 1/2 (voxel
// centres at s), and the ray covers length L = h |d| / |d_A| (= ray_step) in every slab.
// Inside a slab the in-plane cell coordinate Y = fh + 1/2 and the z cell coordinate
// Z = fz + 1/2 are linear in the slab parameter t in [0, 1] (t = 0 at s - 1/2) and move by
// |fhd| <= 1 and |vr Wd| <= 1 (not z-dominant), so the slab's chord crosses at most one
// y and one z cell boundary.  With (ja, ka) the cells at t = 0 and cy, cz in [0, 1] the
// parameters of the crossings (the distance to the next boundary in the direction of
// motion over the distance moved, clamped: 1 = no crossing), the four cells' weights are
//    (ja, ka): min(cy, cz)         (ja, ka + sz): cy - min(cy, cz)
//    (ja + sy, ka): cz - min       (ja + sy, ka + sz): 1 - max(cy, cz)
// (sy, sz = +-1 the directions of motion), times L.  Positions at t = 0 use the anchored
// f32 model above with the +1/2 cell shift folded into the fp64 anchors, so the forward and
// the transpose evaluate identical expressions (bit-identical weights).  Summed over slabs
// this is exactly the 3-D box chord of tests/oracles.hpp:89-107 per voxel.
__device__ __forceinline__ void sid_anchor(const double4& c, int sc, int& jA, float& tA, double& G) {
    dsplit(__dadd_rn(__fma_rn(double(sc), c.y, c.x), 0.5), jA, tA);
    G = __fma_rn(double(sc), c.w, c.z);
}
// z cell coordinate Z = fz + 1/2 = izs + fcs + vr W
__device__ __forceinline__ int sid_izc(const KGeom& g) { return g.nzg >> 1; }
__device__ __forceinline__ float sid_fc(const KGeom& g) { return (g.nzg & 1) ? 0.5f : 0.f; }
// crossing parameter of a cell coordinate with fraction f moving by d per slab: the distance
// to the next boundary in the direction of motion over |d|, clamped to [0, 1] -- one
// saturated FMA, c = sat(f * A + B) with (A, B) = (-1/|d|, 1/|d|) moving up, (1/|d|, 0) down;
// 1/|d| is capped at 1e30 (d = 0: never crosses)
__device__ __forceinline__ float2 sid_coef(bool inc, float ad) {
    ad = fminf(ad, 1e30f);
    return inc ? make_float2(-ad, ad) : make_float2(ad, 0.f);
}
__device__ __forceinline__ float sid_cross(float f, float2 ab) { return __saturatef(fmaf(f, ab.x, ab.y)); }

}  // namespace
}  // namespace ctkb
