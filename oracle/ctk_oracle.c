/*
 * oracle/ctk_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker, never shipped).
 *
 * Plain-C restatement of the reference projector family of `ctkrylov`
 * (/root/reference/proj/include/ctkrylov/projector.hpp, gradient.hpp, tv.hpp,
 * phantom.hpp).  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load this library, and only as the checker.
 *
 * Parity pin: tests/test_oracle.py checks every entry point here bitwise against
 * the reference headers compiled unmodified into oracle/_ref (oracle/ref_capi.cpp)
 * and against the reference's own known-answer tests (test_operators.cpp).
 *
 * Arithmetic is written to reproduce the reference's IEEE operation sequence
 * exactly (compile with -ffp-contract=off, no -march=native): every expression keeps
 * the reference's association order, so T=double results are bit-identical.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int mode;            /* 0 parallel2d, 1 parallel3d, 2 cone3d (geometry.hpp:11) */
    double dso, dod, du; /* source_to_origin, origin_to_detector, pixel size (geometry.hpp:25-28) */
    int nu, nv;
    int nx, ny, nz;
    double h;            /* isotropic voxel spacing (types.hpp:37) */
    int na;
    const double* angles;
} orc_geom;

static const double ORC_TWO_PI = 2.0 * 3.14159265358979323846;

/* canonical_angle, types.hpp:172-177 */
double orc_canonical_angle(double a) {
    double r = fmod(a, ORC_TWO_PI);
    if (r < 0.0) r += ORC_TWO_PI;
    return r;
}

/* ConeGeometry::validate, geometry.hpp:35-54.  Returns 0 ok, 2 geometry error. */
int orc_validate(const orc_geom* g) {
    if (g->na < 1) return 2;
    if (g->nu <= 0 || g->nv <= 0) return 2;
    if (!(g->du > 0.0)) return 2;
    if (!(g->dod > 0.0)) return 2;
    if (g->nx <= 0 || g->ny <= 0 || g->nz <= 0 || !(g->h > 0.0)) return 2;
    if (g->mode == 0 && (g->nz != 1 || g->nv != 1)) return 2;
    if (g->mode == 2) {
        if (!(g->dso > 0.0)) return 2;
        double hx = 0.5 * g->nx * g->h, hy = 0.5 * g->ny * g->h, hz = 0.5 * g->nz * g->h;
        double half_diag = sqrt(hx * hx + hy * hy + hz * hz);
        if (g->dso <= half_diag) return 2;
    }
    return 0;
}

/* ---- ray model: make_ray (projector.hpp:29-46) + plan_walk (projector.hpp:48-91) ---- */
typedef struct {
    int axis, n_slices, nb, nc;
    double step, fb0, fb_d, fc0, fc_d;
    size_t sa, sb, sc;
} orc_walk;

static void orc_make_walk(const orc_geom* g, double ct, double st, int iu, int iv, orc_walk* w) {
    double o[3], d[3];
    const double u = (iu - 0.5 * (g->nu - 1)) * g->du;
    const double v = (iv - 0.5 * (g->nv - 1)) * g->du;
    const double cx = -g->dod * ct, cy = -g->dod * st, cz = 0.0;
    const double px = cx - u * st, py = cy + u * ct, pz = cz + v;
    if (g->mode == 2) {
        const double sx = g->dso * ct, sy = g->dso * st, sz = 0.0;
        double dx = px - sx, dy = py - sy, dz = pz - sz;
        const double n = sqrt(dx * dx + dy * dy + dz * dz);
        o[0] = sx; o[1] = sy; o[2] = sz;
        d[0] = dx / n; d[1] = dy / n; d[2] = dz / n;
    } else {
        o[0] = px; o[1] = py; o[2] = pz;
        d[0] = -ct; d[1] = -st; d[2] = 0.0;
    }
    const double ad[3] = {fabs(d[0]), fabs(d[1]), fabs(d[2])};
    int axis = 0;
    if (ad[1] > ad[axis]) axis = 1;
    if (ad[2] > ad[axis]) axis = 2;
    const int n3[3] = {g->nx, g->ny, g->nz};
    const size_t s3[3] = {1, (size_t)g->nx, (size_t)g->nx * (size_t)g->ny};
    const int b = (axis + 1) % 3, c = (axis + 2) % 3;
    const double h = g->h;
    w->axis = axis;
    w->n_slices = n3[axis];
    w->step = h / ad[axis];
    w->nb = n3[b];
    w->nc = n3[c];
    w->sa = s3[axis];
    w->sb = s3[b];
    w->sc = s3[c];
    const double t0 = ((0 - 0.5 * (n3[axis] - 1)) * h - o[axis]) / d[axis];
    const double dt = h / d[axis];
    w->fb0 = (o[b] + t0 * d[b]) / h + 0.5 * (n3[b] - 1);
    w->fb_d = dt * d[b] / h;
    w->fc0 = (o[c] + t0 * d[c]) / h + 0.5 * (n3[c] - 1);
    w->fc_d = dt * d[c] / h;
}

/* for_slice_stencil (projector.hpp:93-111): up to four (index, weight) pairs in fixed order */
static int orc_stencil(const orc_walk* w, int s, size_t idx[4], double wgt[4]) {
    const double fb = w->fb0 + s * w->fb_d;
    const double fc = w->fc0 + s * w->fc_d;
    const int ib = (int)floor(fb);
    const int ic = (int)floor(fc);
    const double tb = fb - ib, tc = fc - ic;
    const size_t base = w->sa * (size_t)s;
    const double wq[4] = {(1 - tb) * (1 - tc), tb * (1 - tc), (1 - tb) * tc, tb * tc};
    int m = 0;
    for (int q = 0; q < 4; ++q) {
        const int jb = ib + (q & 1), jc = ic + (q >> 1);
        if (jb < 0 || jb >= w->nb || jc < 0 || jc >= w->nc || wq[q] == 0.0) continue;
        idx[m] = base + w->sb * (size_t)jb + w->sc * (size_t)jc;
        wgt[m] = wq[q];
        ++m;
    }
    return m;
}

/* T-generic bodies; T = double and float.  Mirrors integrate_ray (projector.hpp:113-122),
 * forward_project (:134-162), scatter_ray (:124-130), back_project_matched (:166-202),
 * back_project_voxel_driven (:204-279). */
#define ORC_DEFINE(T, SUF)                                                                     \
    void orc_forward_##SUF(const orc_geom* g, const T* vol, T* proj) {                         \
        const size_t frame = (size_t)g->nu * g->nv;                                            \
        for (int a = 0; a < g->na; ++a) {                                                      \
            const double th = orc_canonical_angle(g->angles[a]);                               \
            const double ct = cos(th), st = sin(th);                                           \
            for (int iv = 0; iv < g->nv; ++iv)                                                 \
                for (int iu = 0; iu < g->nu; ++iu) {                                           \
                    orc_walk w;                                                                \
                    orc_make_walk(g, ct, st, iu, iv, &w);                                      \
                    T acc = 0;                                                                 \
                    for (int s = 0; s < w.n_slices; ++s) {                                     \
                        size_t idx[4];                                                         \
                        double wt[4];                                                          \
                        const int m = orc_stencil(&w, s, idx, wt);                             \
                        T sample = 0;                                                          \
                        for (int q = 0; q < m; ++q) sample += (T)wt[q] * vol[idx[q]];          \
                        acc += sample;                                                         \
                    }                                                                          \
                    proj[(size_t)a * frame + (size_t)iu + (size_t)g->nu * iv] = (T)w.step * acc; \
                }                                                                              \
        }                                                                                      \
    }                                                                                          \
                                                                                               \
    /* nparts = the reference's OpenMP thread count (min(omp_max_threads, n_angles)); the     \
     * partial volumes are accumulated and summed in the same order (projector.hpp:172-201). */ \
    void orc_back_matched_##SUF(const orc_geom* g, const T* proj, T* vol, int nparts) {       \
        const size_t nvox = (size_t)g->nx * g->ny * g->nz;                                     \
        const size_t frame = (size_t)g->nu * g->nv;                                            \
        if (nparts < 1) nparts = 1;                                                            \
        if (nparts > g->na) nparts = g->na;                                                    \
        T* part = (T*)malloc(nvox * sizeof(T));                                                \
        for (size_t i = 0; i < nvox; ++i) vol[i] = 0;                                          \
        for (int t = 0; t < nparts; ++t) {                                                     \
            memset(part, 0, nvox * sizeof(T));                                                 \
            for (int a = t; a < g->na; a += nparts) {                                          \
                const double th = orc_canonical_angle(g->angles[a]);                           \
                const double ct = cos(th), st = sin(th);                                       \
                for (int iv = 0; iv < g->nv; ++iv)                                             \
                    for (int iu = 0; iu < g->nu; ++iu) {                                       \
                        const T value = proj[(size_t)a * frame + (size_t)iu + (size_t)g->nu * iv]; \
                        if (value == (T)0) continue;                                           \
                        orc_walk w;                                                            \
                        orc_make_walk(g, ct, st, iu, iv, &w);                                  \
                        const T scaled = (T)w.step * value;                                    \
                        for (int s = 0; s < w.n_slices; ++s) {                                 \
                            size_t idx[4];                                                     \
                            double wt[4];                                                      \
                            const int m = orc_stencil(&w, s, idx, wt);                         \
                            for (int q = 0; q < m; ++q) part[idx[q]] += (T)wt[q] * scaled;     \
                        }                                                                      \
                    }                                                                          \
            }                                                                                  \
            for (size_t i = 0; i < nvox; ++i) vol[i] += (T)1 * part[i];                        \
        }                                                                                      \
        free(part);                                                                            \
    }                                                                                          \
                                                                                               \
    void orc_back_voxel_##SUF(const orc_geom* g, const T* proj, T* vol) {                      \
        const size_t frame = (size_t)g->nu * g->nv;                                            \
        double* ct = (double*)malloc(sizeof(double) * g->na);                                  \
        double* st = (double*)malloc(sizeof(double) * g->na);                                  \
        double* sc = (double*)malloc(sizeof(double) * g->na);                                  \
        for (int a = 0; a < g->na; ++a) {                                                      \
            const double th = orc_canonical_angle(g->angles[a]);                               \
            ct[a] = cos(th);                                                                   \
            st[a] = sin(th);                                                                   \
            sc[a] = 0.0;                                                                       \
            if (g->mode != 2) {                                                                \
                const double m = fmax(fabs(ct[a]), fabs(st[a]));                               \
                sc[a] = g->h / m;                                                              \
            }                                                                                  \
        }                                                                                      \
        for (int k = 0; k < g->nz; ++k) {                                                      \
            const double z = (k - 0.5 * (g->nz - 1)) * g->h;                                   \
            for (int j = 0; j < g->ny; ++j) {                                                  \
                const double y = (j - 0.5 * (g->ny - 1)) * g->h;                               \
                for (int i = 0; i < g->nx; ++i) {                                              \
                    const double x = (i - 0.5 * (g->nx - 1)) * g->h;                           \
                    T acc = 0;                                                                 \
                    for (int a = 0; a < g->na; ++a) {                                          \
                        double u, v, scale;                                                    \
                        if (g->mode == 2) {                                                    \
                            const double sx = g->dso * ct[a], sy = g->dso * st[a];             \
                            const double rx = x - sx, ry = y - sy, rz = z;                     \
                            const double depth = -(rx * ct[a] + ry * st[a]);                   \
                            if (depth <= 0.0) continue;                                        \
                            const double t = (g->dso + g->dod) / depth;                        \
                            const double px = sx + t * rx, py = sy + t * ry, pz = t * rz;      \
                            u = -px * st[a] + py * ct[a];                                      \
                            v = pz;                                                            \
                            const double rn = sqrt(rx * rx + ry * ry + rz * rz);               \
                            const double dom = fmax(fabs(rx), fmax(fabs(ry), fabs(rz)));       \
                            scale = g->h * rn / dom;                                           \
                        } else {                                                               \
                            u = -x * st[a] + y * ct[a];                                        \
                            v = z;                                                             \
                            scale = sc[a];                                                     \
                        }                                                                      \
                        const double fu = u / g->du + 0.5 * (g->nu - 1);                       \
                        const double fv = (g->nv == 1) ? 0.0 : v / g->du + 0.5 * (g->nv - 1);  \
                        const int iu = (int)floor(fu), iv = (int)floor(fv);                    \
                        const double tu = fu - iu, tv = fv - iv;                               \
                        const T* fr = proj + (size_t)a * frame;                                \
                        double sample = 0.0;                                                   \
                        const double wq[4] = {(1 - tu) * (1 - tv), tu * (1 - tv), (1 - tu) * tv, tu * tv}; \
                        for (int q = 0; q < 4; ++q) {                                          \
                            const int ju = iu + (q & 1), jv = iv + (q >> 1);                   \
                            if (ju < 0 || ju >= g->nu || jv < 0 || jv >= g->nv) continue;      \
                            sample += wq[q] * (double)fr[(size_t)ju + (size_t)g->nu * jv];     \
                        }                                                                      \
                        acc += (T)(scale * sample);                                            \
                    }                                                                          \
                    vol[(size_t)i + (size_t)g->nx * ((size_t)j + (size_t)g->ny * k)] = acc;    \
                }                                                                              \
            }                                                                                  \
        }                                                                                      \
        free(ct);                                                                              \
        free(st);                                                                              \
        free(sc);                                                                              \
    }                                                                                          \
                                                                                               \
    /* gradient (gradient.hpp:9-27): forward differences, zero on the far face */             \
    void orc_gradient_##SUF(int nx, int ny, int nz, const T* v, T* dx, T* dy, T* dz) {         \
        for (int k = 0; k < nz; ++k)                                                           \
            for (int j = 0; j < ny; ++j)                                                       \
                for (int i = 0; i < nx; ++i) {                                                 \
                    const size_t id = (size_t)i + (size_t)nx * ((size_t)j + (size_t)ny * k);   \
                    dx[id] = (i + 1 < nx) ? v[id + 1] - v[id] : (T)0;                          \
                    dy[id] = (j + 1 < ny) ? v[id + (size_t)nx] - v[id] : (T)0;                 \
                    dz[id] = (k + 1 < nz) ? v[id + (size_t)nx * ny] - v[id] : (T)0;            \
                }                                                                              \
    }                                                                                          \
                                                                                               \
    /* gradient_adjoint (gradient.hpp:29-54): exact transpose, fixed term order */             \
    void orc_gradient_adjoint_##SUF(int nx, int ny, int nz, const T* dx, const T* dy,          \
                                    const T* dz, T* out) {                                     \
        const size_t sy = (size_t)nx, sz = (size_t)nx * ny;                                    \
        for (int k = 0; k < nz; ++k)                                                           \
            for (int j = 0; j < ny; ++j)                                                       \
                for (int i = 0; i < nx; ++i) {                                                 \
                    const size_t id = (size_t)i + sy * ((size_t)j + (size_t)ny * k);           \
                    T acc = 0;                                                                 \
                    if (i > 0) acc += dx[id - 1];                                              \
                    if (i + 1 < nx) acc -= dx[id];                                             \
                    if (j > 0) acc += dy[id - sy];                                             \
                    if (j + 1 < ny) acc -= dy[id];                                             \
                    if (k > 0) acc += dz[id - sz];                                             \
                    if (k + 1 < nz) acc -= dz[id];                                             \
                    out[id] = acc;                                                             \
                }                                                                              \
    }                                                                                          \
                                                                                               \
    /* tv_weights (tv.hpp:17-43): w = (|Dx|^2 + eps^2)^(-1/4), eps = 1e-4 max|x| */            \
    void orc_tv_weights_##SUF(int nx, int ny, int nz, const T* x, T* w) {                      \
        const size_t n = (size_t)nx * ny * nz;                                                 \
        double m = 0.0;                                                                        \
        for (size_t i = 0; i < n; ++i) m = fmax(m, fabs((double)x[i]));                        \
        const double eps = 1e-4 * m;                                                           \
        if (eps == 0.0) {                                                                      \
            for (size_t i = 0; i < n; ++i) w[i] = (T)1;                                        \
            return;                                                                            \
        }                                                                                      \
        T* gx = (T*)malloc(n * sizeof(T));                                                     \
        T* gy = (T*)malloc(n * sizeof(T));                                                     \
        T* gz = (T*)malloc(n * sizeof(T));                                                     \
        orc_gradient_##SUF(nx, ny, nz, x, gx, gy, gz);                                         \
        for (size_t i = 0; i < n; ++i) {                                                       \
            const double m2 = (double)gx[i] * gx[i] + (double)gy[i] * gy[i] + (double)gz[i] * gz[i]; \
            w[i] = (T)pow(m2 + eps * eps, -0.25);                                              \
        }                                                                                      \
        free(gx);                                                                              \
        free(gy);                                                                              \
        free(gz);                                                                              \
    }

ORC_DEFINE(double, f64)
ORC_DEFINE(float, f32)

/* ---- Siddon exact-length projector (new: absent from the reference).
 * Ray geometry = make_ray (projector.hpp:29-46).  Voxel (i,j,k) is the box
 * [(i - n/2) h, (i + 1 - n/2) h] x ... (centres at (i - (n-1)/2) h, types.hpp:50).  The
 * weight of (ray, voxel) is the length of the ray inside the voxel box, i.e. the slab
 * chord of tests/oracles.hpp:89-107 applied to that voxel.  Every plane crossing is
 * evaluated as alpha_a(q) = ((q - n_a/2) h - o_a) * inv_a with inv_a = 1/d_a, both by the
 * forward DDA and by the transpose, so the two see bit-identical segment lengths.  A ray
 * parallel to an axis belongs to the half-open slab [plane q, plane q+1) containing o_a. */
typedef struct {
    double o[3], d[3], inv[3];
} orc_ray;

static void orc_make_ray(const orc_geom* g, double ct, double st, int iu, int iv, orc_ray* r) {
    const double u = (iu - 0.5 * (g->nu - 1)) * g->du;
    const double v = (iv - 0.5 * (g->nv - 1)) * g->du;
    const double cx = -g->dod * ct, cy = -g->dod * st, cz = 0.0;
    const double px = cx - u * st, py = cy + u * ct, pz = cz + v;
    if (g->mode == 2) {
        const double sx = g->dso * ct, sy = g->dso * st, sz = 0.0;
        const double dx = px - sx, dy = py - sy, dz = pz - sz;
        const double n = sqrt(dx * dx + dy * dy + dz * dz);
        r->o[0] = sx; r->o[1] = sy; r->o[2] = sz;
        r->d[0] = dx / n; r->d[1] = dy / n; r->d[2] = dz / n;
    } else {
        r->o[0] = px; r->o[1] = py; r->o[2] = pz;
        r->d[0] = -ct; r->d[1] = -st; r->d[2] = 0.0;
    }
    for (int a = 0; a < 3; ++a) r->inv[a] = r->d[a] != 0.0 ? 1.0 / r->d[a] : 0.0;
}

static double orc_plane_alpha(const orc_ray* r, int a, int q, int n, double h) {
    return ((q - 0.5 * n) * h - r->o[a]) * r->inv[a];
}

/* slab index of a coordinate: floor((c - lo) / h) with lo = -n h / 2 */
static int orc_slab(double c, int n, double h) { return (int)floor(c / h + 0.5 * n); }

/* chord of ray r inside voxel idx3 (0 if it misses) */
static double orc_voxel_chord(const orc_ray* r, const int n3[3], double h, const int idx3[3]) {
    double lo = -INFINITY, hi = INFINITY;
    for (int a = 0; a < 3; ++a) {
        if (r->d[a] == 0.0) {
            if (orc_slab(r->o[a], n3[a], h) != idx3[a]) return 0.0;
            continue;
        }
        const double a0 = orc_plane_alpha(r, a, idx3[a], n3[a], h);
        const double a1 = orc_plane_alpha(r, a, idx3[a] + 1, n3[a], h);
        lo = fmax(lo, fmin(a0, a1));
        hi = fmin(hi, fmax(a0, a1));
    }
    return hi > lo ? hi - lo : 0.0;
}

/* DDA over the voxels the ray crosses; calls fn(idx, length) in traversal order */
#define ORC_SIDDON_WALK(g, r, BODY)                                                         \
    do {                                                                                     \
        const int n3_[3] = {(g)->nx, (g)->ny, (g)->nz};                                      \
        const double h_ = (g)->h;                                                            \
        double amin_ = -INFINITY, amax_ = INFINITY;                                          \
        int ok_ = 1;                                                                         \
        for (int a_ = 0; a_ < 3 && ok_; ++a_) {                                              \
            if ((r).d[a_] == 0.0) {                                                          \
                const int s_ = orc_slab((r).o[a_], n3_[a_], h_);                             \
                if (s_ < 0 || s_ >= n3_[a_]) ok_ = 0;                                        \
                continue;                                                                    \
            }                                                                                \
            const double e0_ = orc_plane_alpha(&(r), a_, 0, n3_[a_], h_);                    \
            const double e1_ = orc_plane_alpha(&(r), a_, n3_[a_], n3_[a_], h_);              \
            amin_ = fmax(amin_, fmin(e0_, e1_));                                             \
            amax_ = fmin(amax_, fmax(e0_, e1_));                                             \
        }                                                                                    \
        if (ok_ && amin_ < amax_) {                                                          \
            int ix_[3], st_[3];                                                              \
            double an_[3];                                                                   \
            for (int a_ = 0; a_ < 3; ++a_) {                                                 \
                if ((r).d[a_] == 0.0) {                                                      \
                    ix_[a_] = orc_slab((r).o[a_], n3_[a_], h_);                              \
                    st_[a_] = 0;                                                             \
                    an_[a_] = INFINITY;                                                      \
                    continue;                                                                \
                }                                                                            \
                st_[a_] = (r).d[a_] > 0.0 ? 1 : -1;                                          \
                /* voxel entered at amin: the slab whose entry plane crossing is <= amin */  \
                int q_ = st_[a_] > 0 ? 0 : n3_[a_] - 1;                                       \
                while (1) {                                                                  \
                    const double ax_ = orc_plane_alpha(&(r), a_, st_[a_] > 0 ? q_ + 1 : q_, n3_[a_], h_); \
                    if (ax_ > amin_ || (st_[a_] > 0 ? q_ == n3_[a_] - 1 : q_ == 0)) break;  \
                    q_ += st_[a_];                                                           \
                }                                                                            \
                ix_[a_] = q_;                                                                \
                an_[a_] = orc_plane_alpha(&(r), a_, st_[a_] > 0 ? q_ + 1 : q_, n3_[a_], h_); \
            }                                                                                \
            double acur_ = amin_;                                                            \
            while (acur_ < amax_) {                                                          \
                double anext_ = fmin(amax_, fmin(an_[0], fmin(an_[1], an_[2])));             \
                const double len_ = anext_ - acur_;                                          \
                const size_t idx_ = (size_t)ix_[0] + (size_t)n3_[0] * ((size_t)ix_[1] + (size_t)n3_[1] * ix_[2]); \
                if (len_ > 0.0) { BODY }                                                     \
                if (anext_ >= amax_) break;                                                  \
                int out_ = 0;                                                                \
                for (int a_ = 0; a_ < 3; ++a_)                                               \
                    if (an_[a_] == anext_) {                                                 \
                        ix_[a_] += st_[a_];                                                  \
                        if (ix_[a_] < 0 || ix_[a_] >= n3_[a_]) out_ = 1;                     \
                        an_[a_] = orc_plane_alpha(&(r), a_, st_[a_] > 0 ? ix_[a_] + 1 : ix_[a_], n3_[a_], h_); \
                    }                                                                        \
                if (out_) break;                                                             \
                acur_ = anext_;                                                              \
            }                                                                                \
        }                                                                                    \
    } while (0)

#define ORC_SIDDON_DEFINE(T, SUF)                                                               \
    void orc_siddon_forward_##SUF(const orc_geom* g, const T* vol, T* proj) {                  \
        const size_t frame = (size_t)g->nu * g->nv;                                            \
        for (int a = 0; a < g->na; ++a) {                                                      \
            const double th = orc_canonical_angle(g->angles[a]);                               \
            const double ct = cos(th), st = sin(th);                                           \
            for (int iv = 0; iv < g->nv; ++iv)                                                 \
                for (int iu = 0; iu < g->nu; ++iu) {                                           \
                    orc_ray r;                                                                 \
                    orc_make_ray(g, ct, st, iu, iv, &r);                                       \
                    T acc = 0;                                                                 \
                    ORC_SIDDON_WALK(g, r, { acc += (T)len_ * vol[idx_]; });                    \
                    proj[(size_t)a * frame + (size_t)iu + (size_t)g->nu * iv] = acc;           \
                }                                                                              \
        }                                                                                      \
    }                                                                                          \
    /* exact transpose as a scatter in (angle, iv, iu, traversal) order */                     \
    void orc_siddon_back_##SUF(const orc_geom* g, const T* proj, T* vol) {                     \
        const size_t frame = (size_t)g->nu * g->nv;                                            \
        const size_t nvox = (size_t)g->nx * g->ny * g->nz;                                     \
        for (size_t i = 0; i < nvox; ++i) vol[i] = 0;                                          \
        for (int a = 0; a < g->na; ++a) {                                                      \
            const double th = orc_canonical_angle(g->angles[a]);                               \
            const double ct = cos(th), st = sin(th);                                           \
            for (int iv = 0; iv < g->nv; ++iv)                                                 \
                for (int iu = 0; iu < g->nu; ++iu) {                                           \
                    const T value = proj[(size_t)a * frame + (size_t)iu + (size_t)g->nu * iv]; \
                    if (value == (T)0) continue;                                               \
                    orc_ray r;                                                                 \
                    orc_make_ray(g, ct, st, iu, iv, &r);                                       \
                    ORC_SIDDON_WALK(g, r, { vol[idx_] += (T)len_ * value; });                  \
                }                                                                              \
        }                                                                                      \
    }

ORC_SIDDON_DEFINE(double, f64)
ORC_SIDDON_DEFINE(float, f32)

/* chord of one ray with one voxel (both in the conventions above), for the tests */
double orc_siddon_chord(const orc_geom* g, int a, int iu, int iv, int i, int j, int k) {
    const double th = orc_canonical_angle(g->angles[a]);
    orc_ray r;
    orc_make_ray(g, cos(th), sin(th), iu, iv, &r);
    const int n3[3] = {g->nx, g->ny, g->nz}, idx3[3] = {i, j, k};
    return orc_voxel_chord(&r, n3, g->h, idx3);
}

/* Walk description of one ray, exposed so tests can pin the kernels' per-ray setup
 * (axis, step, affine slice indices) against the restated plan_walk. */
void orc_walk_params(const orc_geom* g, int a, int iu, int iv, int* axis, double out5[5]) {
    const double th = orc_canonical_angle(g->angles[a]);
    orc_walk w;
    orc_make_walk(g, cos(th), sin(th), iu, iv, &w);
    *axis = w.axis;
    out5[0] = w.step;
    out5[1] = w.fb0;
    out5[2] = w.fb_d;
    out5[3] = w.fc0;
    out5[4] = w.fc_d;
}

/* Shepp-Logan 3D rasteriser (phantom.hpp:74-145): ten ellipsoids, cell-centre sampling. */
static const double ORC_SL3D[10][8] = {
    {0.0, 0.0, 0.0, 0.69, 0.92, 0.81, 0.0, 2.0},
    {0.0, -0.0184, 0.0, 0.6624, 0.874, 0.78, 0.0, -0.8},
    {0.22, 0.0, 0.0, 0.11, 0.31, 0.22, -18.0, -0.2},
    {-0.22, 0.0, 0.0, 0.16, 0.41, 0.28, 18.0, -0.2},
    {0.0, 0.35, -0.15, 0.21, 0.25, 0.41, 0.0, 0.1},
    {0.0, 0.1, 0.25, 0.046, 0.046, 0.05, 0.0, 0.1},
    {0.0, -0.1, 0.25, 0.046, 0.046, 0.05, 0.0, 0.1},
    {-0.08, -0.605, 0.0, 0.046, 0.023, 0.05, 0.0, 0.1},
    {0.0, -0.605, 0.0, 0.023, 0.023, 0.02, 0.0, 0.1},
    {0.06, -0.605, 0.0, 0.023, 0.046, 0.02, 0.0, 0.1},
};

void orc_shepp_logan_3d_f64(int n, double* out) {
    const double pi = 3.14159265358979323846;
    for (int k = 0; k < n; ++k) {
        const double z = n == 1 ? 0.0 : (double)(2 * k + 1 - n) / n;
        for (int j = 0; j < n; ++j) {
            const double y = (double)(2 * j + 1 - n) / n;
            for (int i = 0; i < n; ++i) {
                const double x = (double)(2 * i + 1 - n) / n;
                double v = 0.0;
                for (int e = 0; e < 10; ++e) {
                    const double* p = ORC_SL3D[e];
                    const double phi = p[6] * pi / 180.0;
                    const double c = cos(phi), s = sin(phi);
                    const double ddx = x - p[0], ddy = y - p[1], ddz = z - p[2];
                    const double xr = c * ddx + s * ddy;
                    const double yr = -s * ddx + c * ddy;
                    const double uu = xr / p[3], vv = yr / p[4], ww = ddz / p[5];
                    if (uu * uu + vv * vv + ww * ww <= 1.0) v += p[7];
                }
                out[(size_t)i + (size_t)n * ((size_t)j + (size_t)n * k)] = v;
            }
        }
    }
}
