// Geometry handle: validation (ConeGeometry::validate, geometry.hpp:35-54), canonical
// angles (types.hpp:172-177), host-libm cos/sin per view (make_ray, projector.hpp:33),
// and the per-(view, column) f32 ray tables of the separable model (kernels_f32.cu).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <numbers>

#include "ctk_internal.h"

namespace ctkb {

static std::atomic<uint64_t> g_launches{0};
uint64_t launch_count() { return g_launches.load(); }

void after_launch(const char* what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(CTK_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

DevBuf::~DevBuf() { release(); }
void DevBuf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
}
bool DevBuf::ensure(size_t nbytes) {
    if (nbytes <= bytes && p) return false;
    release();
    if (nbytes == 0) nbytes = 16;
    CTK_CUDA(cudaMalloc(&p, nbytes));
    bytes = nbytes;
    return true;
}

KGeom Geometry::kgeom() const {
    KGeom k;
    k.mode = mode;
    k.nu = nu;
    k.nv = nv;
    k.nx = nx;
    k.ny = ny;
    k.nz = nz_local();
    k.nzg = nz;
    k.z0 = slab ? z0 : 0;
    k.w0 = band ? w0 : 0;
    k.nw = band ? nw : nv;
    k.na = na;
    k.has_zrays = has_zrays ? 1 : 0;
    k.dso = dso;
    k.dod = dod;
    k.du = du;
    k.h = h;
    k.ctst = d_ctst.as<double2>();
    k.col = d_col.as<float4>();
    k.col64 = d_col64.as<double4>();
    k.colaxis = d_colaxis.as<unsigned char>();
    k.vclass = d_vclass.as<int4>();
    k.colstep = d_colstep.as<double2>();
#ifdef CTK_CHECKED
    k.chk = d_chk.as<unsigned>();
#endif
    return k;
}

void Geometry::require_angles() const {
    if (!angles_valid) fail(CTK_E_GEOMETRY, angles_msg);
}

Geometry::~Geometry() {
    if (pinned) cudaFreeHost(pinned);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (own_stream && stream) cudaStreamDestroy(stream);
}

static double canonical_angle(double a) {
    constexpr double two_pi = 2.0 * std::numbers::pi;
    double r = std::fmod(a, two_pi);
    if (r < 0.0) r += two_pi;
    return r;
}

void geometry_validate(const ctk_geom_desc* d) {
    if (!d) fail(CTK_E_PARAMETER, "null geometry descriptor");
    // ConeGeometry::validate, in the reference's order and wording
    if (d->n_angles <= 0 || !d->angles) fail(CTK_E_GEOMETRY, "geometry needs at least one angle");
    if (d->nu <= 0 || d->nv <= 0) fail(CTK_E_GEOMETRY, "detector pixel counts must be positive");
    if (!(d->detector_pixel_size > 0.0)) fail(CTK_E_GEOMETRY, "detector pixel size must be positive");
    if (!(d->origin_to_detector > 0.0)) fail(CTK_E_GEOMETRY, "origin-to-detector distance must be positive");
    if (d->nx <= 0 || d->ny <= 0 || d->nz <= 0 || !(d->spacing > 0.0))
        fail(CTK_E_GEOMETRY, "geometry volume descriptor invalid");
    if (d->mode < 0 || d->mode > 2) fail(CTK_E_PARAMETER, "unknown beam mode");
    if (d->mode == CTK_PARALLEL2D && (d->nz != 1 || d->nv != 1))
        fail(CTK_E_GEOMETRY, "parallel2d requires nz = 1 and nv = 1");
    if (d->mode == CTK_CONE3D) {
        if (!(d->source_to_origin > 0.0)) fail(CTK_E_GEOMETRY, "cone3d requires a positive source-to-origin distance");
        const double hx = 0.5 * d->nx * d->spacing, hy = 0.5 * d->ny * d->spacing, hz = 0.5 * d->nz * d->spacing;
        const double half_diag = std::sqrt(hx * hx + hy * hy + hz * hz);
        if (d->source_to_origin <= half_diag) fail(CTK_E_GEOMETRY, "cone3d source lies inside the volume diagonal");
    }
}

Geometry* geometry_create(const ctk_geom_desc* d) {
    geometry_validate(d);

    auto* g = new Geometry();
    try {
        g->mode = d->mode;
        g->nu = d->nu;
        g->nv = d->nv;
        g->nx = d->nx;
        g->ny = d->ny;
        g->nz = d->nz;
        g->na = d->n_angles;
        g->dso = d->source_to_origin;
        g->dod = d->origin_to_detector;
        g->du = d->detector_pixel_size;
        g->h = d->spacing;
        g->angles.resize(size_t(g->na));
        g->ct.resize(size_t(g->na));
        g->st.resize(size_t(g->na));
        for (int a = 0; a < g->na; ++a) {
            // projector_pair canonicalises the captured angles (operators.hpp:96)
            const double th = canonical_angle(d->angles[a]);
            g->angles[size_t(a)] = th;
            g->ct[size_t(a)] = std::cos(th);
            g->st[size_t(a)] = std::sin(th);
        }
        // ProjectionSet::validate (types.hpp:104-117) runs on every apply in the reference
        for (int a = 0; a < g->na; ++a) {
            const double th = g->angles[size_t(a)];
            if (!(th >= 0.0 && th < 2.0 * std::numbers::pi)) {
                g->angles_valid = false;
                g->angles_msg = "angles must lie in [0, 2*pi)";
                break;
            }
            if (a > 0 && !(th > g->angles[size_t(a - 1)])) {
                g->angles_valid = false;
                g->angles_msg = "angles must be strictly increasing";
                break;
            }
        }

        CTK_CUDA(cudaGetDevice(&g->device));
        CTK_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
        g->own_stream = true;
        CTK_CUDA(cudaEventCreate(&g->ev0));
        CTK_CUDA(cudaEventCreate(&g->ev1));
        CTK_CUDA(cudaMallocHost(&g->pinned, sizeof(double) * 64));

        // per-view (cos, sin)
        std::vector<double2> ctst(size_t(g->na));
        for (int a = 0; a < g->na; ++a) ctst[size_t(a)] = make_double2(g->ct[size_t(a)], g->st[size_t(a)]);
        // per-(view, column) separable ray model, fp64 -> f32
        const size_t ncol = size_t(g->na) * g->nu;
        std::vector<float4> col(ncol);
        std::vector<double4> col64(ncol);
        std::vector<unsigned char> cax(ncol);
        std::vector<double2> cst(ncol);
        const double h = g->h;
        const double vmax = 0.5 * (g->nv - 1) * g->du;
        for (int a = 0; a < g->na; ++a) {
            const double ct = g->ct[size_t(a)], st = g->st[size_t(a)];
            for (int iu = 0; iu < g->nu; ++iu) {
                const double u = (iu - 0.5 * (g->nu - 1)) * g->du;
                const double px = -g->dod * ct - u * st, py = -g->dod * st + u * ct;
                double ox, oy, dx, dy;
                if (g->mode == CTK_CONE3D) {
                    ox = g->dso * ct;
                    oy = g->dso * st;
                    dx = px - ox;
                    dy = py - oy;
                } else {
                    ox = px;
                    oy = py;
                    dx = -ct;
                    dy = -st;
                }
                const int A = (std::abs(dy) > std::abs(dx)) ? 1 : 0;
                double fh0, fhd, g0, gd, dA;
                if (A == 0) {
                    const double t0 = (-0.5 * (g->nx - 1) * h - ox) / dx;
                    fh0 = (oy + t0 * dy) / h + 0.5 * (g->ny - 1);
                    fhd = dy / dx;
                    g0 = t0 / h;
                    gd = 1.0 / dx;
                    dA = std::abs(dx);
                } else {
                    const double t0 = (-0.5 * (g->ny - 1) * h - oy) / dy;
                    fh0 = (ox + t0 * dx) / h + 0.5 * (g->nx - 1);
                    fhd = dx / dy;
                    g0 = t0 / h;
                    gd = 1.0 / dy;
                    dA = std::abs(dy);
                }
                if (g->mode != CTK_CONE3D) {  // parallel: z = v along the whole ray
                    g0 = 1.0 / h;
                    gd = 0.0;
                }
                const size_t c = size_t(a) * g->nu + iu;
                col[c] = make_float4(float(fh0), float(fhd), float(g0), float(gd));
                col64[c] = make_double4(fh0, fhd, g0, gd);
                cax[c] = (unsigned char)A;
                cst[c] = make_double2(dx * dx + dy * dy, dA);
                if (g->mode == CTK_CONE3D && vmax > dA) g->has_zrays = true;
            }
        }
        // view visiting order of the forward kernel: x-dominant views (majority of their
        // columns) first, each group in angle order
        std::vector<int> vorder;
        for (int pass = 0; pass < 2; ++pass)
            for (int a = 0; a < g->na; ++a) {
                int nxd = 0;
                for (int iu = 0; iu < g->nu; ++iu) nxd += cax[size_t(a) * g->nu + iu] == 0;
                if ((2 * nxd >= g->nu) == (pass == 0)) vorder.push_back(a);
            }
        // per view and ray class, the hull of that class's detector columns (empty: lo > hi)
        std::vector<int4> vcls(size_t(g->na), make_int4(g->nu, -1, g->nu, -1));
        for (int a = 0; a < g->na; ++a)
            for (int iu = 0; iu < g->nu; ++iu) {
                int4& h = vcls[size_t(a)];
                if (cax[size_t(a) * g->nu + iu] == 0) {
                    h.x = std::min(h.x, iu);
                    h.y = std::max(h.y, iu);
                } else {
                    h.z = std::min(h.z, iu);
                    h.w = std::max(h.w, iu);
                }
            }
        g->d_vclass.ensure(sizeof(int4) * vcls.size());
#ifdef CTK_CHECKED
        g->d_chk.ensure(sizeof(unsigned));
        CTK_CUDA(cudaMemset(g->d_chk.p, 0, sizeof(unsigned)));
#endif
        CTK_CUDA(cudaMemcpy(g->d_vclass.p, vcls.data(), sizeof(int4) * vcls.size(), cudaMemcpyHostToDevice));
        g->d_vorder.ensure(sizeof(int) * vorder.size());
        CTK_CUDA(cudaMemcpy(g->d_vorder.p, vorder.data(), sizeof(int) * vorder.size(), cudaMemcpyHostToDevice));
        g->d_ctst.ensure(sizeof(double2) * ctst.size());
        g->d_col.ensure(sizeof(float4) * col.size());
        g->d_col64.ensure(sizeof(double4) * col64.size());
        CTK_CUDA(cudaMemcpy(g->d_col64.p, col64.data(), sizeof(double4) * col64.size(), cudaMemcpyHostToDevice));
        g->d_colaxis.ensure(cax.size());
        g->d_colstep.ensure(sizeof(double2) * cst.size());
        CTK_CUDA(cudaMemcpy(g->d_ctst.p, ctst.data(), sizeof(double2) * ctst.size(), cudaMemcpyHostToDevice));
        CTK_CUDA(cudaMemcpy(g->d_col.p, col.data(), sizeof(float4) * col.size(), cudaMemcpyHostToDevice));
        CTK_CUDA(cudaMemcpy(g->d_colaxis.p, cax.data(), cax.size(), cudaMemcpyHostToDevice));
        CTK_CUDA(cudaMemcpy(g->d_colstep.p, cst.data(), sizeof(double2) * cst.size(), cudaMemcpyHostToDevice));
    } catch (...) {
        delete g;
        throw;
    }
    return g;
}

RedWork red_work(Geometry* g) {
    const size_t need = sizeof(double) * (size_t(kRedBlocks) * kRedSlots + kRedSlots + 4096 * 2);
    g->red.ensure(need);
    RedWork w;
    w.partials = g->red.as<double>();
    w.results = w.partials + size_t(kRedBlocks) * kRedSlots;
    return w;
}

}  // namespace ctkb
