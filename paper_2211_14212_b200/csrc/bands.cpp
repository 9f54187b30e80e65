// Band-sharded range of z-slab sharding: which detector rows a
// slab's rays reach, the partition of the rows into owned blocks, and the two neighbour
// exchanges of a sharded operator application.
//
//  * reached rows T_r: a cone ray through row coordinate v meets height z at depth d (from
//    the source) where z = v d / (DSO + DOD), and the volume spans depths DSO -+ R (R: the
//    in-plane half-diagonal), so slab r is seen only by the rows between its edges' images at
//    the nearest and farthest depth (parallel beams: v = z), plus the taps' margins;
//  * owned rows O_r: consecutive blocks in rank order covering [0, nv), the boundary between
//    r-1 and r at the image of the slab boundary through the volume centre (magnification
//    (DSO + DOD) / DSO), clamped into T_{r-1} and T_r where they overlap;
//  * held rows L_r = T_r u O_r: a rank's range vectors are [view][L_r][nu], rows of L_r it
//    does not own kept at zero, so range-space reductions over the local vector are the
//    owned rows' and sum over ranks (rank order) to the whole-range value.
// A x: every rank projects its slab onto T_r; the rows of T_r owned by q are sent to q, and
// q sums the partials of its rows in rank order (deterministic).  A^T b: every rank needs
// the values of all of T_r, so owners send their rows of T_r to r (halo broadcast).  Per
// rank memory: N_vox / G + n_angles * |L_r| * nu, i.e. the domain and range both sharded.
#include <algorithm>
#include <cmath>
#include <vector>

#include "ctk_internal.h"

namespace ctkb {

void slab_rows(int mode, int nx, int ny, int nz, int nv, double h, double du, double dso, double dod, int z0, int n,
               int& r0, int& r1) {
    r0 = 0;
    r1 = nv;
    if (nv == 1) return;
    const double cz = 0.5 * (nz - 1);
    const double zlo = (z0 - 2.0 - cz) * h, zhi = (z0 + n + 1.0 - cz) * h;  // taps + margin
    double vlo = zlo, vhi = zhi;
    if (mode == CTK_CONE3D) {
        const double R = 0.5 * h * std::sqrt(double(nx) * nx + double(ny) * ny) + 2.0 * h;
        if (!(dso - R > 0.0)) return;
        const double D = dso + dod, dn = dso - R, df = dso + R;
        vlo = std::min(zlo * D / dn, zlo * D / df);
        vhi = std::max(zhi * D / dn, zhi * D / df);
    }
    const double cv = 0.5 * (nv - 1);
    r0 = std::max(0, int(std::floor(vlo / du + cv)) - 2);
    r1 = std::min(nv, int(std::ceil(vhi / du + cv)) + 3);
    if (r1 < r0) r1 = r0;
}

void slab_rows(const Geometry& g, int z0, int n, int& r0, int& r1) {
    slab_rows(g.mode, g.nx, g.ny, g.nz, g.nv, g.h, g.du, g.dso, g.dod, z0, n, r0, r1);
}

void band_partition(int mode, int nx, int ny, int nz, int nv, double h, double du, double dso, double dod, int nranks,
                    const int* z0s, const int* ns, int* t0, int* t1, int* o0, int* o1) {
    if (nranks < 1) fail(CTK_E_PARAMETER, "band partition: nranks must be >= 1");
    for (int r = 0; r < nranks; ++r) {
        const int expect = r == 0 ? 0 : z0s[r - 1] + ns[r - 1];
        if (z0s[r] != expect || ns[r] < 1) fail(CTK_E_PARAMETER, "band partition: slabs must tile z in rank order");
        slab_rows(mode, nx, ny, nz, nv, h, du, dso, dod, z0s[r], ns[r], t0[r], t1[r]);
    }
    if (z0s[nranks - 1] + ns[nranks - 1] != nz) fail(CTK_E_PARAMETER, "band partition: slabs must cover the volume");
    const double cz = 0.5 * (nz - 1), cv = 0.5 * (nv - 1);
    const double mag = mode == CTK_CONE3D ? (dso + dod) / dso : 1.0;
    o0[0] = 0;
    for (int r = 1; r < nranks; ++r) {
        const double zb = (z0s[r] - 0.5 - cz) * h;  // the plane between slices z0_r - 1 and z0_r
        int b = int(std::floor(zb * mag / du + cv + 0.5));
        if (t0[r] <= t1[r - 1]) b = std::min(std::max(b, t0[r]), t1[r - 1]);
        b = std::min(std::max(b, o0[r - 1]), nv);
        o1[r - 1] = b;
        o0[r] = b;
    }
    o1[nranks - 1] = nv;
}

namespace {
struct Seg {
    int peer, r0, r1;  // global rows [r0, r1)
    size_t off;        // element offset in the staging buffer
};
size_t seg_elems(const Geometry& g, const Seg& s) { return size_t(g.na) * size_t(s.r1 - s.r0) * g.nu; }

// rows [r0, r1) of every view of a held-row vector <-> a packed [na][r1 - r0][nu] block
template <class T>
void copy_rows(const Geometry& g, T* packed, T* local, int r0, int r1, bool pack, cudaStream_t s) {
    const size_t w = sizeof(T) * size_t(r1 - r0) * g.nu, lp = sizeof(T) * size_t(g.nw) * g.nu;
    T* lrow = local + size_t(r0 - g.w0) * g.nu;
    if (pack) CTK_CUDA(cudaMemcpy2DAsync(packed, w, lrow, lp, w, size_t(g.na), cudaMemcpyDeviceToDevice, s));
    else CTK_CUDA(cudaMemcpy2DAsync(lrow, lp, packed, w, w, size_t(g.na), cudaMemcpyDeviceToDevice, s));
}
}  // namespace

template <class T>
void band_reduce(Geometry& g, T* y, cudaStream_t s) {
    const int R = g.comm->cb.nranks, me = g.comm->cb.rank;
    if (R > 32) fail(CTK_E_UNSUPPORTED, "band-sharded range: at most 32 ranks");
    std::vector<Seg> sends, recvs;
    size_t ns = 0, nr = 0;
    for (int q = 0; q < R; ++q) {
        if (q == me) continue;
        const int a0 = std::max(g.bt0[me], g.bo0[q]), a1 = std::min(g.bt1[me], g.bo1[q]);  // my partial of q's rows
        if (a1 > a0) { sends.push_back({q, a0, a1, ns}); ns += seg_elems(g, sends.back()); }
        const int b0 = std::max(g.bt0[q], g.bo0[me]), b1 = std::min(g.bt1[q], g.bo1[me]);  // q's partial of mine
        if (b1 > b0) { recvs.push_back({q, b0, b1, nr}); nr += seg_elems(g, recvs.back()); }
    }
    g.band_send.ensure(sizeof(T) * std::max<size_t>(ns, 1));
    g.band_recv.ensure(sizeof(T) * std::max<size_t>(nr, 1));
    std::vector<ctk_p2p_op> ops;
    for (const Seg& sg : sends) {
        copy_rows<T>(g, g.band_send.as<T>() + sg.off, y, sg.r0, sg.r1, true, s);
        ops.push_back({sg.peer, 1, g.band_send.as<T>() + sg.off, seg_elems(g, sg)});
    }
    for (const Seg& sg : recvs) ops.push_back({sg.peer, 0, g.band_recv.as<T>() + sg.off, seg_elems(g, sg)});
    comm_exchange(g.comm, ops, sizeof(T) == 8 ? 1 : 0, s);
    // y's owned rows <- sum over ranks in rank order of the partials; the other held rows <- 0
    BandSum<T> bs{};
    bs.n = 0;
    bs.o0 = g.bo0[me];
    bs.o1 = g.bo1[me];
    for (int r = 0; r < R; ++r) {
        if (r == me) {
            bs.src[bs.n++] = {y, std::max(g.bt0[me], g.w0), std::min(g.bt1[me], g.w0 + g.nw), g.nw, g.w0};
            continue;
        }
        for (const Seg& sg : recvs)
            if (sg.peer == r) bs.src[bs.n++] = {g.band_recv.as<T>() + sg.off, sg.r0, sg.r1, sg.r1 - sg.r0, sg.r0};
    }
    band_sum<T>(g, bs, y, s);
}

template <class T>
const T* band_halo(Geometry& g, const T* y, cudaStream_t s) {
    const int R = g.comm->cb.nranks, me = g.comm->cb.rank;
    g.band_scratch.ensure(sizeof(T) * g.range());
    T* out = g.band_scratch.as<T>();
    CTK_CUDA(cudaMemcpyAsync(out, y, sizeof(T) * g.range(), cudaMemcpyDeviceToDevice, s));
    std::vector<Seg> sends, recvs;
    size_t ns = 0, nr = 0;
    for (int q = 0; q < R; ++q) {
        if (q == me) continue;
        const int a0 = std::max(g.bo0[me], g.bt0[q]), a1 = std::min(g.bo1[me], g.bt1[q]);  // my rows q reaches
        if (a1 > a0) { sends.push_back({q, a0, a1, ns}); ns += seg_elems(g, sends.back()); }
        const int b0 = std::max(g.bo0[q], g.bt0[me]), b1 = std::min(g.bo1[q], g.bt1[me]);  // q's rows I reach
        if (b1 > b0) { recvs.push_back({q, b0, b1, nr}); nr += seg_elems(g, recvs.back()); }
    }
    if (sends.empty() && recvs.empty()) return out;
    g.band_send.ensure(sizeof(T) * std::max<size_t>(ns, 1));
    g.band_recv.ensure(sizeof(T) * std::max<size_t>(nr, 1));
    std::vector<ctk_p2p_op> ops;
    for (const Seg& sg : sends) {
        copy_rows<T>(g, g.band_send.as<T>() + sg.off, const_cast<T*>(y), sg.r0, sg.r1, true, s);
        ops.push_back({sg.peer, 1, g.band_send.as<T>() + sg.off, seg_elems(g, sg)});
    }
    for (const Seg& sg : recvs) ops.push_back({sg.peer, 0, g.band_recv.as<T>() + sg.off, seg_elems(g, sg)});
    comm_exchange(g.comm, ops, sizeof(T) == 8 ? 1 : 0, s);
    for (const Seg& sg : recvs) copy_rows<T>(g, g.band_recv.as<T>() + sg.off, out, sg.r0, sg.r1, false, s);
    return out;
}

template void band_reduce<float>(Geometry&, float*, cudaStream_t);
template void band_reduce<double>(Geometry&, double*, cudaStream_t);
template const float* band_halo<float>(Geometry&, const float*, cudaStream_t);
template const double* band_halo<double>(Geometry&, const double*, cudaStream_t);

}  // namespace ctkb
