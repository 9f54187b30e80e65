// Exact-parity kernels for T = double (compiled with --fmad=false so no a*b+c is
// contracted).  Every expression keeps the reference's association order, cos/sin come
// from the host libm, and the per-voxel accumulation order of the matched transpose is
// the reference's (angle partition, angle, iv, iu) order -- so the results are
// bit-identical to the reference's T=double CPU path:
//   forward_project            projector.hpp:134-162 (make_ray :29-46, plan_walk :60-91,
//                              for_slice_stencil :96-111, integrate_ray :113-122)
//   back_project_matched       projector.hpp:166-202 as a deterministic GATHER
//   back_project_voxel_driven  projector.hpp:204-279
#include <cfloat>

#include "ctk_internal.h"

namespace ctkb {
namespace {

struct Walk {
    int axis, n_slices, nb, nc;
    double step, fb0, fb_d, fc0, fc_d;
    size_t sa, sb, sc;
};

// make_ray + plan_walk, operation for operation.
__device__ __forceinline__ void make_walk(const KGeom& g, double ct, double st, int iu, int iv, Walk& w) {
    double o[3], d[3];
    const double u = (iu - 0.5 * (g.nu - 1)) * g.du;
    const double v = (iv - 0.5 * (g.nv - 1)) * g.du;
    const double cx = -g.dod * ct, cy = -g.dod * st, cz = 0.0;
    const double px = cx - u * st, py = cy + u * ct, pz = cz + v;
    if (g.mode == CTK_CONE3D) {
        const double sx = g.dso * ct, sy = g.dso * st, sz = 0.0;
        const double dx = px - sx, dy = py - sy, dz = pz - sz;
        const double n = sqrt(dx * dx + dy * dy + dz * dz);
        o[0] = sx; o[1] = sy; o[2] = sz;
        d[0] = dx / n; d[1] = dy / n; d[2] = dz / n;
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
    const size_t s3[3] = {1, size_t(g.nx), size_t(g.nx) * size_t(g.ny)};
    const int b = axis == 2 ? 0 : axis + 1, c = axis == 0 ? 2 : axis - 1;
    const double h = g.h;
    w.axis = axis;
    w.n_slices = n3[axis];
    w.step = h / adm;
    w.nb = n3[b];
    w.nc = n3[c];
    w.sa = s3[axis];
    w.sb = s3[b];
    w.sc = s3[c];
    const double t0 = ((0 - 0.5 * (n3[axis] - 1)) * h - o[axis]) / d[axis];
    const double dt = h / d[axis];
    w.fb0 = (o[b] + t0 * d[b]) / h + 0.5 * (n3[b] - 1);
    w.fb_d = dt * d[b] / h;
    w.fc0 = (o[c] + t0 * d[c]) / h + 0.5 * (n3[c] - 1);
    w.fc_d = dt * d[c] / h;
}

// Conservative slice range [s0, s1] outside of which no tap of the stencil is inside the
// volume (f in (lo, hi) is required on both in-plane axes).  Skipped slices would add an
// exact +0.0 to the running sum, so clipping does not change a single bit.
__device__ __forceinline__ void clip_axis(double f0, double fd, double lo, double hi, int& s0, int& s1) {
    if (fd == 0.0) {
        if (!(f0 > lo - 1.0 && f0 < hi + 1.0)) { s0 = 1; s1 = 0; }
        return;
    }
    double a = (lo - f0) / fd, b = (hi - f0) / fd;
    if (a > b) { const double t = a; a = b; b = t; }
    if (a > 2e9 || b < -2e9) { s0 = 1; s1 = 0; return; }
    const double lo_s = fmax(a, -2e9), hi_s = fmin(b, 2e9);
    s0 = max(s0, int(floor(lo_s)) - 1);
    s1 = min(s1, int(ceil(hi_s)) + 1);
}

// forward_project (projector.hpp:134-162): thread per ray, make_walk + the slice loop
// operation for operation; lanes along detector ROWS and z-fastest copies of the volume, so
// a warp's taps are consecutive in memory: x-dominant rays read X[i][j][k] (slice i, b = y,
// c = z), y-dominant rays Y[j][i][k] (slice j, b = z, c = x), z-dominant rays the original
// x[k][j][i].  Only the strides change -- the taps, weights, skips and summation order are
// make_walk's, so the result is bit-identical to the reference.
__global__ void k_ax_exact_zfast(KGeom g, const double* __restrict__ vol, const double* __restrict__ vx,
                                 const double* __restrict__ vy, double* __restrict__ proj) {
    const int iv = blockIdx.x * blockDim.x + threadIdx.x;
    const int iu = blockIdx.y * blockDim.y + threadIdx.y;
    const int a = blockIdx.z;
    if (iu >= g.nu || iv >= g.nv) return;
    const double2 cs = g.ctst[a];
    Walk w;
    make_walk(g, cs.x, cs.y, iu, iv, w);
    const double* src = vol;
    if (w.axis == 0) {
        src = vx;
        w.sa = size_t(g.ny) * g.nz; w.sb = size_t(g.nz); w.sc = 1;
    } else if (w.axis == 1) {
        src = vy;
        w.sa = size_t(g.nx) * g.nz; w.sb = 1; w.sc = size_t(g.nz);
    }
    int s0 = 0, s1 = w.n_slices - 1;
    clip_axis(w.fb0, w.fb_d, -1.0, double(w.nb), s0, s1);
    clip_axis(w.fc0, w.fc_d, -1.0, double(w.nc), s0, s1);
    double acc = 0;
    for (int s = s0; s <= s1; ++s) {
        const double fb = w.fb0 + s * w.fb_d;
        const double fc = w.fc0 + s * w.fc_d;
        const int ib = int(floor(fb));
        const int ic = int(floor(fc));
        const double tb = fb - ib, tc = fc - ic;
        const size_t base = w.sa * size_t(s);
        const double wq[4] = {(1 - tb) * (1 - tc), tb * (1 - tc), (1 - tb) * tc, tb * tc};
        double sample = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int jb = ib + (q & 1), jc = ic + (q >> 1);
            if (jb < 0 || jb >= w.nb || jc < 0 || jc >= w.nc || wq[q] == 0.0) continue;
            sample += wq[q] * __ldg(src + base + w.sb * size_t(jb) + w.sc * size_t(jc));
        }
        acc += sample;
    }
    proj[size_t(a) * g.nu * g.nv + size_t(iu) + size_t(g.nu) * iv] = w.step * acc;
}

// x[k][j][i] -> X[i][j][k] and Y[j][i][k] (32 x 32 (i, k) tile transposes per j)
__global__ void k_relayout_f64(int nx, int ny, int nz, const double* __restrict__ x, double* __restrict__ X,
                               double* __restrict__ Y) {
    __shared__ double tile[32][33];
    const int i0 = blockIdx.x * 32, k0 = blockIdx.y * 32, j = blockIdx.z;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int i = i0 + threadIdx.x, k = k0 + r;
        tile[r][threadIdx.x] = (i < nx && k < nz) ? x[size_t(i) + size_t(nx) * (j + size_t(ny) * k)] : 0.0;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int i = i0 + r, k = k0 + threadIdx.x;
        if (i < nx && k < nz) {
            const double v = tile[threadIdx.x][r];
            X[(size_t(i) * ny + j) * nz + k] = v;
            Y[(size_t(j) * nx + i) * nz + k] = v;
        }
    }
}

// Projection of a point onto continuous detector coordinates (fu, fv); false when the
// point is not strictly in front of the cone source (then every pixel is a candidate).
__device__ __forceinline__ bool project_point(const KGeom& g, double ct, double st, double x, double y,
                                              double z, double& fu, double& fv) {
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

// plan_walk of every ray, once per geometry: {axis, fb0, fb_d, fc0, fc_d, step}, so the
// transpose's candidates cost a 48-byte load instead of make_ray's sqrt and divisions.
// Layout [a][iu][iv] (detector columns contiguous, as the gather's lanes read them).
__global__ void k_walk_table(KGeom g, double* __restrict__ tab) {
    const int iu = blockIdx.x * blockDim.x + threadIdx.x;
    const int iv = blockIdx.y * blockDim.y + threadIdx.y;
    const int a = blockIdx.z;
    if (iu >= g.nu || iv >= g.nv) return;
    const double2 cs = g.ctst[a];
    Walk w;
    make_walk(g, cs.x, cs.y, iu, iv, w);
    double* o = tab + 6 * ((size_t(a) * g.nu + iu) * g.nv + iv);
    o[0] = double(w.axis);
    o[1] = w.fb0;
    o[2] = w.fb_d;
    o[3] = w.fc0;
    o[4] = w.fc_d;
    o[5] = w.step;
}

// Exact transpose as a gather, warp = 32 consecutive z voxels of one (i, j) column: voxel
// (i,j,k) sums w * (step * y) over every ray whose Joseph stencil touches it, in the
// reference's scatter order (angle partition, angle, iv, iu).  A ray touches the voxel only
// if it crosses the cube [voxel +- h]^3 (its stencil point in the voxel's slice lies within
// one voxel of it), i.e. only pixel centres inside the bounding box of the cube's 8 corner
// projections (1e-6-pixel slack) are candidates.  Bit-identical to the scatter: the same
// plan_walk values (tabulated) and the same per-voxel summation order.
__global__ void __launch_bounds__(128) k_atb_matched_exact(KGeom g, int nparts, const double* __restrict__ walk,
                                                           const double* __restrict__ pt, double* __restrict__ vol,
                                                           int kblocks) {
    const long wid = long(blockIdx.x) * blockDim.y + threadIdx.y;
    const long ncol = long(g.nx) * g.ny;
    if (wid >= ncol * kblocks) return;
    const int kb = int(wid / ncol) * 32;
    const long col = wid % ncol;
    const int i = int(col % g.nx), j = int(col / g.nx), k = kb + int(threadIdx.x);
    if (k >= g.nz) return;
    const double h = g.h;
    const double xc = (i - 0.5 * (g.nx - 1)) * h, yc = (j - 0.5 * (g.ny - 1)) * h, zc = (k - 0.5 * (g.nz - 1)) * h;
    const int vidx[3] = {i, j, k};
    const size_t frame = size_t(g.nu) * g.nv;
    const double cu = 0.5 * (g.nu - 1), cvv = 0.5 * (g.nv - 1);
    double out = 0;
    for (int t = 0; t < nparts; ++t) {
        double part = 0;
        for (int a = t; a < g.na; a += nparts) {
            const double2 cs = g.ctst[a];
            // candidate window in f32: only a superset of the touching rays is needed (each
            // candidate is decided by the exact plan_walk test); 1e-2-pixel slack
            float umin = FLT_MAX, umax = -FLT_MAX, vmin = FLT_MAX, vmax = -FLT_MAX;
            bool all = false;
            const float ctf = float(cs.x), stf = float(cs.y), hf = float(h);
            const float zlo = float(zc - h), zhi = float(zc + h);
            for (int q = 0; q < 4; ++q) {  // the cube's 4 (x, y) corners, each with z = zc -+ h
                const float x = float(xc) + ((q & 1) ? hf : -hf), y = float(yc) + ((q & 2) ? hf : -hf);
                float u, tz;
                if (g.mode == CTK_CONE3D) {
                    const float depth = float(g.dso) - (x * ctf + y * stf);
                    if (!(depth > 1e-6f * float(g.dso))) { all = true; break; }
                    tz = float(g.dso + g.dod) * __frcp_rn(depth);
                    u = (-x * stf + y * ctf) * tz;
                } else {
                    tz = 1.f;
                    u = -x * stf + y * ctf;
                }
                umin = fminf(umin, u); umax = fmaxf(umax, u);
                vmin = fminf(vmin, fminf(zlo * tz, zhi * tz));
                vmax = fmaxf(vmax, fmaxf(zlo * tz, zhi * tz));
            }
            int iu0 = 0, iu1 = g.nu - 1, iv0 = 0, iv1 = g.nv - 1;
            if (!all) {
                const float idu = float(1.0 / g.du), epsf = 1e-2f;
                iu0 = max(iu0, int(ceilf(fmaxf(fmaf(umin, idu, float(cu) - epsf), -1e9f))));
                iu1 = min(iu1, int(floorf(fminf(fmaf(umax, idu, float(cu) + epsf), 1e9f))));
                if (g.nv > 1) {
                    iv0 = max(iv0, int(ceilf(fmaxf(fmaf(vmin, idu, float(cvv) - epsf), -1e9f))));
                    iv1 = min(iv1, int(floorf(fminf(fmaf(vmax, idu, float(cvv) + epsf), 1e9f))));
                }
            }
            const double* fa = pt + size_t(a) * frame;
            const double* wa = walk + 6 * size_t(a) * frame;
            for (int iv = iv0; iv <= iv1; ++iv) {
                for (int iu = iu0; iu <= iu1; ++iu) {
                    const size_t q = size_t(iu) * g.nv + iv;  // [a][iu][iv]
                    const double value = __ldg(fa + q);
                    if (value == 0.0) continue;
                    const double* wr = wa + 6 * q;
                    const int axis = int(__ldg(wr));
                    const int s = vidx[axis];
                    const int pb = vidx[axis == 2 ? 0 : axis + 1];
                    const int pc = vidx[axis == 0 ? 2 : axis - 1];
                    const double fb = __ldg(wr + 1) + s * __ldg(wr + 2);
                    const double fc = __ldg(wr + 3) + s * __ldg(wr + 4);
                    const int ib = int(floor(fb));
                    const int ic = int(floor(fc));
                    const int ob = pb - ib, oc = pc - ic;
                    if (ob < 0 || ob > 1 || oc < 0 || oc > 1) continue;
                    const double tb = fb - ib, tc = fc - ic;
                    double wq;
                    switch (ob + 2 * oc) {
                        case 0: wq = (1 - tb) * (1 - tc); break;
                        case 1: wq = tb * (1 - tc); break;
                        case 2: wq = (1 - tb) * tc; break;
                        default: wq = tb * tc; break;
                    }
                    if (wq == 0.0) continue;
                    const double scaled = __ldg(wr + 5) * value;
                    part += wq * scaled;
                }
            }
        }
        out += 1.0 * part;
    }
    vol[size_t(i) + size_t(g.nx) * (size_t(j) + size_t(g.ny) * k)] = out;
}

// y[a][iv][iu] -> pt[a][iu][iv]
__global__ void k_transpose_f64(int nu, int nv, const double* __restrict__ y, double* __restrict__ pt) {
    __shared__ double tile[32][33];
    const int a = blockIdx.z, u0 = blockIdx.x * 32, v0 = blockIdx.y * 32;
    const size_t frame = size_t(nu) * nv;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int iu = u0 + threadIdx.x, iv = v0 + r;
        tile[r][threadIdx.x] = (iu < nu && iv < nv) ? y[a * frame + size_t(iv) * nu + iu] : 0.0;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int iu = u0 + r, iv = v0 + threadIdx.x;
        if (iu < nu && iv < nv) pt[a * frame + size_t(iu) * nv + iv] = tile[threadIdx.x][r];
    }
}

// back_project_voxel_driven, per voxel over views in order (projector.hpp:208-279).
__global__ void k_atb_voxel_exact(KGeom g, const double* __restrict__ scale_par,
                                  const double* __restrict__ proj, double* __restrict__ vol) {
    const size_t nvox = size_t(g.nx) * g.ny * g.nz;
    const size_t id = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (id >= nvox) return;
    const int i = int(id % g.nx);
    const int j = int((id / g.nx) % g.ny);
    const int k = int(id / (size_t(g.nx) * g.ny));
    const double z = (k - 0.5 * (g.nz - 1)) * g.h;
    const double y = (j - 0.5 * (g.ny - 1)) * g.h;
    const double x = (i - 0.5 * (g.nx - 1)) * g.h;
    const size_t frame = size_t(g.nu) * g.nv;
    double acc = 0;
    for (int a = 0; a < g.na; ++a) {
        const double2 cs = g.ctst[a];
        const double ct = cs.x, st = cs.y;
        double u, v, scale;
        if (g.mode == CTK_CONE3D) {
            const double sx = g.dso * ct, sy = g.dso * st;
            const double rx = x - sx, ry = y - sy, rz = z;
            const double depth = -(rx * ct + ry * st);
            if (depth <= 0.0) continue;
            const double t = (g.dso + g.dod) / depth;
            const double px = sx + t * rx, py = sy + t * ry, pz = t * rz;
            u = -px * st + py * ct;
            v = pz;
            const double rn = sqrt(rx * rx + ry * ry + rz * rz);
            const double arx = fabs(rx), ary = fabs(ry), arz = fabs(rz);
            const double m1 = (ary < arz) ? arz : ary;  // std::max(|ry|, |rz|)
            const double dom = (arx < m1) ? m1 : arx;   // std::max(|rx|, m1)
            scale = g.h * rn / dom;
        } else {
            u = -x * st + y * ct;
            v = z;
            scale = scale_par[a];
        }
        const double fu = u / g.du + 0.5 * (g.nu - 1);
        const double fv = (g.nv == 1) ? 0.0 : v / g.du + 0.5 * (g.nv - 1);
        const int iu = int(floor(fu)), iv = int(floor(fv));
        const double tu = fu - iu, tv = fv - iv;
        const double* fr = proj + size_t(a) * frame;
        double sample = 0.0;
        const double wq[4] = {(1 - tu) * (1 - tv), tu * (1 - tv), (1 - tu) * tv, tu * tv};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int ju = iu + (q & 1), jv = iv + (q >> 1);
            if (ju < 0 || ju >= g.nu || jv < 0 || jv >= g.nv) continue;
            sample += wq[q] * __ldg(fr + size_t(ju) + size_t(g.nu) * jv);
        }
        acc += scale * sample;
    }
    vol[id] = acc;
}

}  // namespace

void launch_ax_exact_f64(Geometry& g, const double* x, double* y, cudaStream_t s) {
    const size_t nvox = g.domain();
    g.dx64.ensure(nvox * sizeof(double));
    g.dy64.ensure(nvox * sizeof(double));
    {
        dim3 blk(32, 8), grd((g.nx + 31) / 32, (g.nz + 31) / 32, g.ny);
        k_relayout_f64<<<grd, blk, 0, s>>>(g.nx, g.ny, g.nz, x, g.dx64.as<double>(), g.dy64.as<double>());
        after_launch("k_relayout_f64");
    }
    dim3 blk(32, 4);
    dim3 grd((g.nv + 31) / 32, (g.nu + 3) / 4, g.na);
    k_ax_exact_zfast<<<grd, blk, 0, s>>>(g.kgeom(), x, g.dx64.as<double>(), g.dy64.as<double>(), y);
    after_launch("k_ax_exact_zfast");
}

void launch_atb_matched_exact_f64(Geometry& g, const double* y, double* x, cudaStream_t s) {
    const size_t nrays = g.range();
    dim3 rb(32, 8), rg((g.nu + 31) / 32, (g.nv + 31) / 32, g.na);
    if (g.d_walk.ensure(6 * nrays * sizeof(double)) || !g.walk_ready) {
        dim3 wb(32, 4), wg((g.nu + 31) / 32, (g.nv + 3) / 4, g.na);
        k_walk_table<<<wg, wb, 0, s>>>(g.kgeom(), g.d_walk.as<double>());
        after_launch("k_walk_table");
        g.walk_ready = true;
    }
    g.proj_t.ensure(nrays * sizeof(double));
    k_transpose_f64<<<rg, rb, 0, s>>>(g.nu, g.nv, y, g.proj_t.as<double>());
    after_launch("k_transpose_f64");
    const int nparts = std::max(1, std::min(g.bp_parts, g.na));
    const int kblocks = (g.nz + 31) / 32;
    const long warps = long(g.nx) * g.ny * kblocks;
    k_atb_matched_exact<<<unsigned((warps + 3) / 4), dim3(32, 4), 0, s>>>(g.kgeom(), nparts, g.d_walk.as<double>(),
                                                                        g.proj_t.as<double>(), x, kblocks);
    after_launch("k_atb_matched_exact");
}

void launch_atb_voxel_f64(Geometry& g, const double* y, double* x, cudaStream_t s) {
    if (!g.vscale_ready) {
        // per-view parallel-beam scale h / max(|cos|, |sin|) (projector.hpp:216-222), host libm
        std::vector<double> sc(size_t(g.na), 0.0);
        if (g.mode != CTK_CONE3D)
            for (int a = 0; a < g.na; ++a) {
                const double act = std::abs(g.ct[size_t(a)]), ast = std::abs(g.st[size_t(a)]);
                sc[size_t(a)] = g.h / ((act < ast) ? ast : act);
            }
        g.d_vscale.ensure(sizeof(double) * sc.size());
        CTK_CUDA(cudaMemcpy(g.d_vscale.p, sc.data(), sizeof(double) * sc.size(), cudaMemcpyHostToDevice));
        g.vscale_ready = true;
    }
    const size_t n = g.domain();
    k_atb_voxel_exact<<<unsigned((n + 127) / 128), 128, 0, s>>>(g.kgeom(), g.d_vscale.as<double>(), y, x);
    after_launch("k_atb_voxel_exact");
}

}  // namespace ctkb
