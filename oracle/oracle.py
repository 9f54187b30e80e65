"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY (the parity checker; never the product).

Two CPU oracles for the Ax / A^T b hot path of the reference `ctkrylov`:

* ``Restated`` -- ctypes over ``oracle/libctk_oracle.so``, the plain-C restatement
  (oracle/ctk_oracle.c) of projector.hpp / gradient.hpp / tv.hpp / phantom.hpp, plus the
  numpy restatement of the solver recurrences below (solvers.hpp, hybrid.hpp,
  regparam.hpp, tv.hpp).
* ``Reference`` -- ctypes over ``oracle/_ref/libctkref.so``: the UNMODIFIED reference
  headers compiled by oracle/Makefile (extern "C" shim oracle/ref_capi.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module.  Nothing here is reachable from paper_2211_14212_b200.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libctk_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libctkref.so")

PARALLEL2D, PARALLEL3D, CONE3D = 0, 1, 2
MATCHED, VOXEL_DRIVEN = 0, 1
STOP_REASONS = ("max_iters", "residual_increase", "tolerance", "breakdown")


class _CGeom(C.Structure):
    _fields_ = [
        ("mode", C.c_int),
        ("dso", C.c_double),
        ("dod", C.c_double),
        ("du", C.c_double),
        ("nu", C.c_int),
        ("nv", C.c_int),
        ("nx", C.c_int),
        ("ny", C.c_int),
        ("nz", C.c_int),
        ("h", C.c_double),
        ("na", C.c_int),
        ("angles", C.POINTER(C.c_double)),
    ]


@dataclass
class Geom:
    """Mirror of ctk::ConeGeometry (geometry.hpp:24-55)."""

    mode: int
    dso: float
    dod: float
    du: float
    nu: int
    nv: int
    nx: int
    ny: int
    nz: int
    h: float
    angles: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def cstruct(self):
        ang = np.ascontiguousarray(self.angles, dtype=np.float64)
        s = _CGeom(self.mode, self.dso, self.dod, self.du, self.nu, self.nv, self.nx, self.ny,
                   self.nz, self.h, len(ang), ang.ctypes.data_as(C.POINTER(C.c_double)))
        s._keep = ang  # keep the angle buffer alive with the struct
        return s

    @property
    def na(self):
        return len(self.angles)

    @property
    def domain_size(self):
        return self.nx * self.ny * self.nz

    @property
    def range_size(self):
        return self.na * self.nu * self.nv

    def subset(self, idx):
        return Geom(self.mode, self.dso, self.dod, self.du, self.nu, self.nv, self.nx, self.ny,
                    self.nz, self.h, np.asarray(self.angles)[idx].copy())


def equidistant_angles(n, start=0.0, rng=2.0 * math.pi):
    """geometry.hpp:57-64 (canonicalised like canonical_angle, types.hpp:172-177)."""
    a = np.empty(n)
    for i in range(n):
        r = math.fmod(start + rng * i / n, 2.0 * math.pi)
        a[i] = r + 2.0 * math.pi if r < 0.0 else r
    return a


def bench_geometry(n, na, nuv=None):
    """The configs' cone geometry: DSO=2n, DOD=n, pixel 1.5, nu=nv=n."""
    nuv = n if nuv is None else nuv
    return Geom(CONE3D, 2.0 * n, 1.0 * n, 1.5, nuv, nuv, n, n, n, 1.0, equidistant_angles(na))


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _ct(dtype):
    return C.c_double if np.dtype(dtype) == np.float64 else C.c_float


def _suf(dtype):
    return "f64" if np.dtype(dtype) == np.float64 else "f32"


class Restated:
    """ctypes binding of the plain-C restatement (oracle/ctk_oracle.c)."""

    def __init__(self, path=ORACLE_SO):
        self.lib = C.CDLL(path)
        for s in ("f64", "f32"):
            for nm in ("forward", "back_voxel"):
                getattr(self.lib, f"orc_{nm}_{s}").restype = None
            self.lib[f"orc_back_matched_{s}"].restype = None
        self.lib.orc_canonical_angle.restype = C.c_double
        self.lib.orc_siddon_chord.restype = C.c_double
        self.lib.orc_canonical_angle.argtypes = [C.c_double]

    def forward(self, g: Geom, x):
        x = np.ascontiguousarray(x)
        y = np.zeros(g.range_size, dtype=x.dtype)
        gs = g.cstruct()
        getattr(self.lib, f"orc_forward_{_suf(x.dtype)}")(C.byref(gs), _ptr(x, _ct(x.dtype)), _ptr(y, _ct(x.dtype)))
        return y

    def back(self, g: Geom, y, variant=MATCHED, nparts=1):
        y = np.ascontiguousarray(y)
        x = np.zeros(g.domain_size, dtype=y.dtype)
        gs = g.cstruct()
        ct = _ct(y.dtype)
        if variant == MATCHED:
            getattr(self.lib, f"orc_back_matched_{_suf(y.dtype)}")(C.byref(gs), _ptr(y, ct), _ptr(x, ct), C.c_int(nparts))
        else:
            getattr(self.lib, f"orc_back_voxel_{_suf(y.dtype)}")(C.byref(gs), _ptr(y, ct), _ptr(x, ct))
        return x

    def siddon_forward(self, g: Geom, x):
        """Siddon exact-length Ax (new; chord = tests/oracles.hpp:89-107 per voxel)."""
        x = np.ascontiguousarray(x)
        y = np.zeros(g.range_size, dtype=x.dtype)
        gs = g.cstruct()
        getattr(self.lib, f"orc_siddon_forward_{_suf(x.dtype)}")(C.byref(gs), _ptr(x, _ct(x.dtype)), _ptr(y, _ct(x.dtype)))
        return y

    def siddon_back(self, g: Geom, y):
        """Exact transpose of siddon_forward (scatter in traversal order)."""
        y = np.ascontiguousarray(y)
        x = np.zeros(g.domain_size, dtype=y.dtype)
        gs = g.cstruct()
        getattr(self.lib, f"orc_siddon_back_{_suf(y.dtype)}")(C.byref(gs), _ptr(y, _ct(y.dtype)), _ptr(x, _ct(y.dtype)))
        return x

    def siddon_chord(self, g: Geom, a, iu, iv, i, j, k):
        gs = g.cstruct()
        return self.lib.orc_siddon_chord(C.byref(gs), a, iu, iv, i, j, k)

    def walk(self, g: Geom, a, iu, iv):
        ax = C.c_int()
        out = np.zeros(5)
        gs = g.cstruct()
        self.lib.orc_walk_params(C.byref(gs), C.c_int(a), C.c_int(iu), C.c_int(iv), C.byref(ax), _ptr(out, C.c_double))
        return ax.value, out

    def gradient(self, shape, v):
        nx, ny, nz = shape
        v = np.ascontiguousarray(v)
        ct = _ct(v.dtype)
        d = [np.zeros_like(v) for _ in range(3)]
        getattr(self.lib, f"orc_gradient_{_suf(v.dtype)}")(nx, ny, nz, _ptr(v, ct), *[_ptr(t, ct) for t in d])
        return d

    def gradient_adjoint(self, shape, dx, dy, dz):
        nx, ny, nz = shape
        dx, dy, dz = (np.ascontiguousarray(t) for t in (dx, dy, dz))
        ct = _ct(dx.dtype)
        out = np.zeros_like(dx)
        getattr(self.lib, f"orc_gradient_adjoint_{_suf(dx.dtype)}")(nx, ny, nz, _ptr(dx, ct), _ptr(dy, ct), _ptr(dz, ct), _ptr(out, ct))
        return out

    def tv_weights(self, shape, x):
        nx, ny, nz = shape
        x = np.ascontiguousarray(x)
        ct = _ct(x.dtype)
        w = np.zeros_like(x)
        getattr(self.lib, f"orc_tv_weights_{_suf(x.dtype)}")(nx, ny, nz, _ptr(x, ct), _ptr(w, ct))
        return w

    def shepp_logan_3d(self, n, dtype=np.float32):
        out = np.zeros(n * n * n)
        self.lib.orc_shepp_logan_3d_f64(C.c_int(n), _ptr(out, C.c_double))
        return out.astype(dtype)


class _RefLog(C.Structure):
    _fields_ = [
        ("implicit_residual", C.POINTER(C.c_double)),
        ("explicit_residual", C.POINTER(C.c_double)),
        ("relative_error", C.POINTER(C.c_double)),
        ("lambda_", C.POINTER(C.c_double)),
        ("iterations", C.c_int),
        ("n_relerr", C.c_int),
        ("n_lambda", C.c_int),
        ("iterations_run", C.c_int),
        ("stop_reason", C.c_int),
        ("error_iteration", C.c_int),
        ("outer_starts", C.POINTER(C.c_int)),
        ("n_outer_starts", C.c_int),
        ("stored_domain_basis", C.c_int),
        ("stored_range_basis", C.c_int),
        ("warning_iterations", C.POINTER(C.c_int)),
        ("n_warnings", C.c_int),
    ]


class RefError(RuntimeError):
    def __init__(self, code, iteration=0):
        super().__init__(f"reference raised error code {code}")
        self.code = code
        self.iteration = iteration


SOLVERS = {"cgls": 0, "lsqr": 1, "lsmr": 2, "sirt": 3, "hybrid_lsqr": 4, "cgls_tv": 5, "ab_gmres": 6, "ba_gmres": 7,
           "flsqr_tv": 8}


class Reference:
    """ctypes binding of the unmodified reference (oracle/_ref/libctkref.so)."""

    def __init__(self, path=REF_SO):
        self.lib = C.CDLL(path)
        self.lib.ref_gcv_lambda.restype = C.c_double
        self.lib.ref_dp_lambda.restype = C.c_double
        self.lib.ref_max_threads.restype = C.c_int

    @staticmethod
    def available(path=REF_SO):
        return os.path.exists(path)

    def set_threads(self, n):
        self.lib.ref_set_threads(C.c_int(n))

    def max_threads(self):
        return self.lib.ref_max_threads()

    def forward(self, g: Geom, x):
        x = np.ascontiguousarray(x)
        y = np.zeros(g.range_size, dtype=x.dtype)
        gs = g.cstruct()
        rc = getattr(self.lib, f"ref_forward_{_suf(x.dtype)}")(C.byref(gs), _ptr(x, _ct(x.dtype)), _ptr(y, _ct(x.dtype)))
        if rc:
            raise RefError(rc)
        return y

    def back(self, g: Geom, y, variant=MATCHED):
        y = np.ascontiguousarray(y)
        x = np.zeros(g.domain_size, dtype=y.dtype)
        gs = g.cstruct()
        rc = getattr(self.lib, f"ref_back_{_suf(y.dtype)}")(C.byref(gs), C.c_int(variant), _ptr(y, _ct(y.dtype)), _ptr(x, _ct(y.dtype)))
        if rc:
            raise RefError(rc)
        return x

    def solve(self, g: Geom, b, solver, max_iters, variant=MATCHED, lam=0.0, strategy=0,
              noise_level=0.0, outer=1, inner=1, warm=False, tol=1e-6, stop_inc=True,
              reorth=True, gt=None):
        b = np.ascontiguousarray(b)
        dt = b.dtype
        ct = _ct(dt)
        cap = max(max_iters, outer * inner) + 2
        bufs = [np.zeros(cap) for _ in range(4)]
        outer_buf = np.zeros(outer + 2, dtype=np.int32)
        warn_buf = np.zeros(cap, dtype=np.int32)
        log = _RefLog(*[_ptr(t, C.c_double) for t in bufs], 0, 0, 0, 0, 0, 0,
                      _ptr(outer_buf, C.c_int), 0, 0, 0, _ptr(warn_buf, C.c_int), 0)
        x = np.zeros(g.domain_size, dtype=dt)
        gs = g.cstruct()
        gt_p = None
        if gt is not None:
            gt = np.ascontiguousarray(gt, dtype=dt)
            gt_p = _ptr(gt, ct)
        rc = getattr(self.lib, f"ref_solve_{_suf(dt)}")(
            C.byref(gs), C.c_int(variant), C.c_int(SOLVERS[solver]), C.c_double(lam), C.c_int(strategy),
            C.c_double(noise_level), C.c_int(outer), C.c_int(inner), C.c_int(int(warm)), _ptr(b, ct),
            C.c_int(max_iters), C.c_double(tol), C.c_int(int(stop_inc)), C.c_int(int(reorth)), gt_p,
            _ptr(x, ct), C.byref(log))
        if rc:
            raise RefError(rc, log.error_iteration)
        it = log.iterations
        return {
            "x": x,
            "implicit": bufs[0][:it].copy(),
            "explicit": bufs[1][:it].copy(),
            "relative_error": bufs[2][: log.n_relerr].copy(),
            "lambda": bufs[3][: log.n_lambda].copy(),
            "iterations_run": log.iterations_run,
            "stop_reason": STOP_REASONS[log.stop_reason],
            "outer_starts": outer_buf[: log.n_outer_starts].copy(),
            "stored_domain_basis": log.stored_domain_basis,
            "stored_range_basis": log.stored_range_basis,
            "warning_iterations": warn_buf[: log.n_warnings].copy(),
        }

    def phantom(self, kind, n, dtype=np.float64):
        nz = n if kind == 0 else 1
        out = np.zeros(n * n * nz, dtype=dtype)
        rc = getattr(self.lib, f"ref_phantom_{_suf(dtype)}")(C.c_int(kind), C.c_int(n), _ptr(out, _ct(dtype)))
        if rc:
            raise RefError(rc)
        return out

    def add_noise(self, g: Geom, clean, i0=1e5, sigma=0.5, seed=0):
        clean = np.ascontiguousarray(clean, dtype=np.float64)
        out = np.zeros_like(clean)
        gs = g.cstruct()
        rc = self.lib.ref_add_noise_f64(C.byref(gs), _ptr(clean, C.c_double), C.c_double(i0), C.c_double(sigma),
                                        C.c_uint64(seed), _ptr(out, C.c_double))
        if rc:
            raise RefError(rc)
        return out

    def gcv_lambda(self, H, beta1):
        H = np.ascontiguousarray(H, dtype=np.float64)
        return self.lib.ref_gcv_lambda(_ptr(H, C.c_double), C.c_int(H.shape[1]), C.c_double(beta1))

    def dp_lambda(self, H, beta1, nl):
        H = np.ascontiguousarray(H, dtype=np.float64)
        return self.lib.ref_dp_lambda(_ptr(H, C.c_double), C.c_int(H.shape[1]), C.c_double(beta1), C.c_double(nl))

    def tv_weights(self, shape, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        w = np.zeros_like(x)
        nx, ny, nz = shape
        rc = self.lib.ref_tv_weights_f64(nx, ny, nz, _ptr(x, C.c_double), _ptr(w, C.c_double))
        if rc:
            raise RefError(rc)
        return w


# ---------------------------------------------------------------------------------------
# numpy restatement of the solver recurrences (float64), following solvers.hpp line by line.
# `fwd` / `back` are callables on flat numpy vectors (an OperatorPair, operators.hpp:18-45).
# ---------------------------------------------------------------------------------------
INCREASE_SLACK = 1e-12  # solve_log.hpp:80


class Monitor:
    """IterationMonitor (solve_log.hpp:86-161)."""

    def __init__(self, fwd, b, max_iters, tol, stop_inc, gt=None):
        self.fwd, self.b = fwd, b
        self.bnorm = float(np.linalg.norm(b))
        if not self.bnorm > 0:
            raise ValueError("zero right-hand side")
        self.tol, self.stop_inc, self.gt = tol, stop_inc, gt
        self.gtn = float(np.linalg.norm(gt)) if gt is not None else 0.0
        self.impl, self.expl, self.err, self.lam = [], [], [], []
        self.prev, self.have_prev, self.reason = 0.0, False, "max_iters"

    def record(self, k, x, implicit, lam=None, explicit=None):
        if explicit is None:
            explicit = float(np.linalg.norm(self.fwd(x) - self.b)) / self.bnorm
        if not (math.isfinite(explicit) and math.isfinite(implicit)):
            raise FloatingPointError(f"non-finite residual at iteration {k}")
        self.impl.append(implicit)
        self.expl.append(explicit)
        if lam is not None:
            self.lam.append(lam)
        if self.gt is not None:
            self.err.append(float(np.linalg.norm(x - self.gt)) / self.gtn)
        if explicit <= self.tol:
            self.reason = "tolerance"
            return True
        if self.stop_inc and self.have_prev and explicit > self.prev * (1.0 + INCREASE_SLACK):
            self.reason = "residual_increase"
            return True
        self.prev, self.have_prev = explicit, True
        return False

    def result(self, x, k, **extra):
        d = {"x": x, "implicit": np.array(self.impl), "explicit": np.array(self.expl),
             "relative_error": np.array(self.err), "lambda": np.array(self.lam),
             "iterations_run": k, "stop_reason": self.reason}
        d.update(extra)
        return d


def cgls(fwd, back, b, max_iters, tol=1e-6, stop_inc=True, gt=None):
    """solvers.hpp:13-60."""
    mon = Monitor(fwd, b, max_iters, tol, stop_inc, gt)
    x = np.zeros_like(back(b))
    r = b.copy()
    s = back(r)
    p = s.copy()
    gamma = float(s @ s)
    k = 0
    while k < max_iters:
        k += 1
        if not gamma > 0:
            mon.reason = "breakdown"
            k -= 1
            break
        q = fwd(p)
        delta = float(q @ q)
        if not delta > 0:
            mon.reason = "breakdown"
            k -= 1
            break
        alpha = gamma / delta
        x += alpha * p
        r -= alpha * q
        if mon.record(k, x, float(np.linalg.norm(r)) / mon.bnorm):
            break
        s = back(r)
        gnew = float(s @ s)
        beta = gnew / gamma
        gamma = gnew
        p = s + beta * p
    return mon.result(x, k)


def lsqr(fwd, back, b, max_iters, tol=1e-6, stop_inc=True, gt=None, bd=1e-14):
    """solvers.hpp:62-126."""
    mon = Monitor(fwd, b, max_iters, tol, stop_inc, gt)
    beta1 = float(np.linalg.norm(b))
    tolb = bd * beta1
    u = b / beta1
    v = back(u)
    alpha = float(np.linalg.norm(v))
    v = v / alpha
    w = v.copy()
    x = np.zeros_like(v)
    phibar, rhobar = beta1, alpha
    k = 0
    while k < max_iters:
        k += 1
        unew = fwd(v) - alpha * u
        beta = float(np.linalg.norm(unew))
        down = beta <= tolb
        if beta > 0:
            u = unew / beta
            vnew = back(u) - beta * v
            alpha = float(np.linalg.norm(vnew))
            if alpha > 0:
                v = vnew / alpha
            down = down or alpha <= tolb
        else:
            alpha = 0.0
        rho = math.sqrt(rhobar * rhobar + beta * beta)
        c, s = rhobar / rho, beta / rho
        theta = s * alpha
        rhobar = -c * alpha
        phi = c * phibar
        phibar = s * phibar
        x += (phi / rho) * w
        w = v - (theta / rho) * w
        if mon.record(k, x, phibar / beta1):
            break
        if down:
            mon.reason = "breakdown"
            break
    return mon.result(x, k)


def lsmr(fwd, back, b, lam, max_iters, tol=1e-6, stop_inc=True, gt=None, bd=1e-14):
    """solvers.hpp:128-231 (Fong-Saunders with damping)."""
    mon = Monitor(fwd, b, max_iters, tol, stop_inc, gt)
    damp = lam
    beta1 = float(np.linalg.norm(b))
    tolb = bd * beta1
    u = b / beta1
    v = back(u)
    alpha = float(np.linalg.norm(v))
    v = v / alpha
    zetabar, alphabar = alpha * beta1, alpha
    rho = rhobar = cbar = 1.0
    sbar = 0.0
    h = v.copy()
    hbar = np.zeros_like(v)
    x = np.zeros_like(v)
    betadd, betad, rhodold, tautildeold, thetatilde, zeta, dsq = beta1, 0.0, 1.0, 0.0, 0.0, 0.0, 0.0
    k = 0
    while k < max_iters:
        k += 1
        unew = fwd(v) - alpha * u
        beta = float(np.linalg.norm(unew))
        down = beta <= tolb
        if beta > 0:
            u = unew / beta
            vnew = back(u) - beta * v
            alpha = float(np.linalg.norm(vnew))
            if alpha > 0:
                v = vnew / alpha
            down = down or alpha <= tolb
        else:
            alpha = 0.0
        alphahat = math.sqrt(alphabar * alphabar + damp * damp)
        chat, shat = alphabar / alphahat, damp / alphahat
        rhoold = rho
        rho = math.sqrt(alphahat * alphahat + beta * beta)
        c, s = alphahat / rho, beta / rho
        thetanew = s * alpha
        alphabar = c * alpha
        rhobarold, zetaold = rhobar, zeta
        thetabar = sbar * rho
        rhotemp = cbar * rho
        rhobar = math.sqrt(rhotemp * rhotemp + thetanew * thetanew)
        cbar, sbar = rhotemp / rhobar, thetanew / rhobar
        zeta = cbar * zetabar
        zetabar = -sbar * zetabar
        hbar = h - (thetabar * rho / (rhoold * rhobarold)) * hbar
        x += (zeta / (rho * rhobar)) * hbar
        h = v - (thetanew / rho) * h
        betaacute = chat * betadd
        betacheck = -shat * betadd
        betahat = c * betaacute
        betadd = -s * betaacute
        thetatildeold = thetatilde
        rhotildeold = math.sqrt(rhodold * rhodold + thetabar * thetabar)
        ctildeold, stildeold = rhodold / rhotildeold, thetabar / rhotildeold
        thetatilde = stildeold * rhobar
        rhodold = ctildeold * rhobar
        betad = -stildeold * betad + ctildeold * betahat
        tautildeold = (zetaold - thetatildeold * tautildeold) / rhotildeold
        taud = (zeta - thetatilde * tautildeold) / rhodold
        dsq += betacheck * betacheck
        normr = math.sqrt(dsq + (betad - taud) ** 2 + betadd * betadd)
        if mon.record(k, x, normr / beta1, lam):
            break
        if down:
            mon.reason = "breakdown"
            break
    return mon.result(x, k)


def sirt(fwd, back, b, nd, max_iters, tol=1e-6, stop_inc=True, gt=None):
    """solvers.hpp:233-287: x <- x + C B (R (b - A x)), R / C inverse row / column sums of the
    pair applied to all-ones vectors, floored at 1e-6 of their maximum."""
    if not float(np.linalg.norm(b)) > 0:
        return {"x": np.zeros(nd), "implicit": np.array([]), "explicit": np.array([]), "relative_error": np.array([]),
                "lambda": np.array([]), "iterations_run": 0, "stop_reason": "tolerance"}
    mon = Monitor(fwd, b, max_iters, tol, stop_inc, gt)

    def inverse_weights(w):
        wmax = float(np.max(np.abs(w)))
        if not wmax > 0:
            raise ValueError("sirt: operator maps ones to zero")
        return 1.0 / np.maximum(w, 1e-6 * wmax)

    row_inv = inverse_weights(fwd(np.ones(nd)))
    col_inv = inverse_weights(back(np.ones(b.size)))
    x = np.zeros(nd)
    r = b.copy()
    k = 0
    while k < max_iters:
        k += 1
        x = x + col_inv * back(row_inv * r)
        r = b - fwd(x)
        expl = float(np.linalg.norm(r)) / mon.bnorm
        if mon.record(k, x, expl, explicit=expl):
            break
    return mon.result(x, k)


def abba_gmres(fwd, back, b, max_iters, ab, tol=1e-6, stop_inc=True, gt=None, reorth=True, bd=1e-14):
    """gmres.hpp:41-99 with arnoldi_init/arnoldi_expand (krylov.hpp:94-145): Arnoldi by
    modified Gram-Schmidt (+ a classical second pass when reorth) on A B (AB) or B A (BA);
    projected least squares on the (k+1) x k Hessenberg; x rebuilt from the whole basis."""
    mon = Monitor(fwd, b, max_iters, tol, stop_inc, gt)
    rhs = b.copy() if ab else back(b)
    square = (lambda v: fwd(back(v))) if ab else (lambda v: back(fwd(v)))
    beta1 = float(np.linalg.norm(rhs))
    W = [rhs / beta1]
    hcols = []
    x = None
    k = 0
    while k < max_iters:
        k += 1
        j = len(hcols)
        w = square(W[j])
        h = np.zeros(j + 2)
        for i in range(j + 1):
            h[i] = float(W[i] @ w)
            w = w - h[i] * W[i]
        if reorth:
            for i in range(j + 1):
                c = float(W[i] @ w)
                w = w - c * W[i]
                h[i] += c
        hnext = float(np.linalg.norm(w))
        h[j + 1] = hnext
        hcols.append(h)
        breakdown = hnext <= bd * beta1
        if not breakdown:
            W.append(w / hnext)
        H = np.zeros((k + 1, k))
        for c, col in enumerate(hcols):
            H[: min(len(col), k + 1), c] = col[: k + 1]
        e1 = np.zeros(k + 1)
        e1[0] = beta1
        y = np.linalg.lstsq(H, e1, rcond=None)[0]
        resid = float(np.linalg.norm(e1 - H @ y))
        comb = sum(y[i] * W[i] for i in range(k))
        x = back(comb) if ab else comb
        if mon.record(k, x, resid / beta1):
            break
        if breakdown:
            mon.reason = "breakdown"
            break
    return mon.result(x, k, stored_domain_basis=0 if ab else len(W), stored_range_basis=len(W) if ab else 0)


def gcv_lambda(H, beta1):
    """regparam.hpp:114-159 (linear-convention GCV; 1001-point log scan + golden section)."""
    U, sig, _ = np.linalg.svd(H, full_matrices=False)
    e1 = np.zeros(H.shape[0])
    e1[0] = beta1
    rhs = U.T @ e1
    perp2 = max(0.0, beta1 * beta1 - float(rhs @ rhs))
    k = H.shape[1]

    def gcv(lam):
        s2 = sig * sig
        r = lam / (s2 + lam)
        num = perp2 + float(np.sum((rhs * r) ** 2))
        tr = (k + 1.0) - float(np.sum(s2 / (s2 + lam)))
        return num / (tr * tr)

    smax = sig[0]
    lo, hi = math.log(1e-10 * smax * smax), math.log(1e10 * smax * smax)
    vals = [gcv(math.exp(lo + (hi - lo) * i / 1000)) for i in range(1001)]
    best = int(np.argmin(vals))
    step = (hi - lo) / 1000
    a, b_ = lo + step * max(0, best - 1), lo + step * min(1000, best + 1)
    ip = 0.6180339887498949
    c, d = b_ - ip * (b_ - a), a + ip * (b_ - a)
    fc, fd = gcv(math.exp(c)), gcv(math.exp(d))
    it = 0
    while it < 200 and (b_ - a) > 1e-10:
        if fc < fd:
            b_, d, fd = d, c, fc
            c = b_ - ip * (b_ - a)
            fc = gcv(math.exp(c))
        else:
            a, c, fc = c, d, fd
            d = a + ip * (b_ - a)
            fd = gcv(math.exp(d))
        it += 1
    return math.exp(0.5 * (a + b_))


def dp_lambda(H, beta1, nl):
    """regparam.hpp:79-113 (discrepancy principle by bisection)."""
    U, sig, _ = np.linalg.svd(H, full_matrices=False)
    e1 = np.zeros(H.shape[0])
    e1[0] = beta1
    rhs = U.T @ e1
    perp2 = max(0.0, beta1 * beta1 - float(rhs @ rhs))

    def disc2(lam):
        l2 = lam * lam
        d = sig * sig + l2
        f = np.where(d > 0, l2 / np.where(d > 0, d, 1), 1.0)
        return perp2 + float(np.sum((rhs * f) ** 2))

    target = nl * nl * beta1 * beta1
    if disc2(0.0) >= target * (1.0 - 1e-12):
        return 0.0
    smax = sig[0]
    lo, hi = 1e-10 * smax, 1e10 * smax
    if disc2(lo) >= target:
        a, b_ = 0.0, lo
        for _ in range(200):
            mid = 0.5 * (a + b_)
            d = disc2(mid)
            if abs(d - target) <= 1e-6 * target:
                return mid
            if d < target:
                a = mid
            else:
                b_ = mid
        return 0.5 * (a + b_)
    llo, lhi = math.log(lo), math.log(hi)
    mid = 0.5 * (llo + lhi)
    for _ in range(60):
        mid = 0.5 * (llo + lhi)
        d = disc2(math.exp(mid))
        if abs(d - target) <= 1e-6 * target:
            break
        if d < target:
            llo = mid
        else:
            lhi = mid
    return math.exp(mid)


def projected_tikhonov(H, beta1, lam):
    """hybrid.hpp:37-55."""
    U, sig, Vt = np.linalg.svd(H, full_matrices=False)
    rhs = np.zeros(H.shape[0])
    rhs[0] = beta1
    coef = U.T @ rhs
    d = sig * sig + lam * lam
    yf = np.where(d > 0, sig * coef / np.where(d > 0, d, 1), 0.0)
    y = Vt.T @ yf
    return y, float(np.linalg.norm(rhs - H @ y))


def hybrid_lsqr(fwd, back, b, max_iters, strategy="gcv", lam=0.0, nl=0.0, tol=1e-6, stop_inc=True,
                gt=None, reorth=True, bd=1e-14):
    """hybrid.hpp:76-116 with gk_init/gk_expand (krylov.hpp:50-92) and CGS2 (krylov.hpp:21-31)."""
    mon = Monitor(fwd, b, max_iters, tol, stop_inc, gt)
    beta1 = float(np.linalg.norm(b))
    tolb = bd * beta1
    U = [b / beta1]
    v = back(U[0])
    a1 = float(np.linalg.norm(v))
    V = [v / a1]
    alphas, betas = [a1], []

    def cgs2(basis, w):
        for _ in range(2):
            coef = [float(q @ w) for q in basis]
            for q, c in zip(basis, coef):
                w = w - c * q
        return w

    x = np.zeros_like(V[0])
    k = 0
    while k < max_iters:
        j = len(V)
        status = "ok"
        w = fwd(V[j - 1]) - alphas[j - 1] * U[j - 1]
        if reorth:
            w = cgs2(U, w)
        beta = float(np.linalg.norm(w))
        if beta <= tolb:
            status = "breakdown"
        else:
            U.append(w / beta)
            betas.append(beta)
            z = back(U[j]) - beta * V[j - 1]
            if reorth:
                z = cgs2(V, z)
            alpha = float(np.linalg.norm(z))
            if alpha <= tolb:
                status = "breakdown"
            else:
                V.append(z / alpha)
                alphas.append(alpha)
        if status == "breakdown" and len(betas) < k + 1:
            mon.reason = "breakdown"
            break
        k += 1
        H = np.zeros((k + 1, k))
        for jj in range(k):
            H[jj, jj] = alphas[jj]
            H[jj + 1, jj] = betas[jj]
        if strategy == "fixed":
            lam_k = lam
        elif strategy == "dp":
            lam_k = dp_lambda(H, beta1, nl)
        else:
            lam_k = math.sqrt(max(0.0, gcv_lambda(H, beta1)))
        y, fit = projected_tikhonov(H, beta1, lam_k)
        x = sum(float(y[i]) * V[i] for i in range(len(y)))
        if mon.record(k, x, fit / beta1, lam_k):
            break
        if status == "breakdown":
            mon.reason = "breakdown"
            break
    return mon.result(x, k, stored_domain_basis=len(V), stored_range_basis=len(U))


def flsqr_tv(fwd, back, b, shape, max_iters, restated: Restated, strategy="gcv", lam=0.0, tol=1e-6, stop_inc=True,
             gt=None, reorth=True, bd=1e-14, max_inner=50, inner_tol=1e-6):
    """flsqr_tv (tv.hpp:112-185) = flexible_hybrid_lsqr (hybrid.hpp:118-168) with the TV
    priorconditioner: flexible GK (krylov.hpp:147-224), z_j = CG solve of
    (D^T diag(w^2) D + tau^2 I) z = v_j from zero (tau = 1e-3 lambda0), w = tv_weights(x)."""
    # dots accumulate sequentially like the reference's dot() (types.hpp:137-142): the
    # truncated inner CG amplifies summation-order differences
    def sdot(a, b):
        return float(np.cumsum(a * b)[-1]) if a.size else 0.0

    def snrm(a):
        return math.sqrt(sdot(a, a))

    lambda0 = lam if strategy == "fixed" and lam > 0.0 else 1.0
    tau2 = (1e-3 * lambda0) ** 2
    mon = Monitor(fwd, b, max_iters, tol, stop_inc, gt)
    beta1 = snrm(b)
    tolb = bd * beta1
    U = [b / beta1]
    v = back(U[0])
    V = [v / snrm(v)]
    Z, mcols, warnings = [], [], []
    x = np.zeros_like(V[0])

    def mgs(basis, w, coef=None):
        for i, q in enumerate(basis):
            c = sdot(q, w)
            w = w - c * q
            if coef is not None:
                coef[i] += c
        return w

    k = 0
    while k < max_iters:
        w2 = restated.tv_weights(shape, x) ** 2

        def apply(p):
            dx, dy, dz = restated.gradient(shape, p)
            return restated.gradient_adjoint(shape, w2 * dx, w2 * dy, w2 * dz) + tau2 * p

        j = len(mcols)
        z = np.zeros_like(x)
        r = V[j].copy()
        p = r.copy()
        rr = sdot(r, r)
        target = inner_tol * math.sqrt(rr)
        conv = not math.sqrt(rr) > 0
        for _ in range(max_inner):
            if conv:
                break
            ap = apply(p)
            pap = sdot(p, ap)
            if not pap > 0:
                break
            alpha = rr / pap
            z = z + alpha * p
            r = r - alpha * ap
            rr_new = sdot(r, r)
            if math.sqrt(rr_new) <= target:
                conv = True
                break
            beta = rr_new / rr
            rr = rr_new
            p = r + beta * p
        if not conv:
            warnings.append(k + 1)
        status = "ok"
        if not snrm(z) > 0:
            status = "breakdown"
        else:
            w = fwd(z)
            m = np.zeros(j + 2)
            w = mgs(U, w, m)
            if reorth:
                w = mgs(U, w, m)
            mnext = snrm(w)
            m[j + 1] = mnext
            Z.append(z)
            mcols.append(m)
            if mnext <= tolb:
                status = "breakdown"
            else:
                U.append(w / mnext)
                vn = back(U[-1])
                for _ in range(2 if reorth else 1):
                    vn = mgs(V, vn)
                nv = snrm(vn)
                if nv <= tolb:
                    status = "breakdown"
                else:
                    V.append(vn / nv)
        if status == "breakdown" and len(mcols) < k + 1:
            mon.reason = "breakdown"
            break
        k += 1
        M = np.zeros((k + 1, k))
        for c, col in enumerate(mcols):
            M[: min(len(col), k + 1), c] = col[: k + 1]
        lam_k = lam if strategy == "fixed" else math.sqrt(max(0.0, gcv_lambda(M, beta1)))
        y, fit = projected_tikhonov(M, beta1, lam_k)
        x = sum(float(y[i]) * Z[i] for i in range(len(y)))
        if mon.record(k, x, fit / beta1, lam_k):
            break
        if status == "breakdown":
            mon.reason = "breakdown"
            break
    return mon.result(x, k, stored_domain_basis=len(Z), stored_range_basis=len(U), warnings=warnings)


def cgls_tv(fwd, back, b, shape, lam, outer, inner, restated: Restated, tol=1e-6, stop_inc=True,
            gt=None, warm=False):
    """tv.hpp:45-110 with stack_weighted_gradient (operators.hpp:141-186)."""
    mon = Monitor(fwd, b, outer * inner, tol, stop_inc, gt)
    nvox = int(np.prod(shape))
    nr = b.size
    x = np.zeros(nvox)
    starts = []
    k = 0
    stopped = False
    for _ in range(outer):
        if stopped:
            break
        w = restated.tv_weights(shape, x)

        def sf(xx, w=w):
            gx, gy, gz = restated.gradient(shape, xx)
            return np.concatenate([fwd(xx), lam * w * gx, lam * w * gy, lam * w * gz])

        def sb(yy, w=w):
            s = lam * w
            return back(yy[:nr]) + restated.gradient_adjoint(shape, s * yy[nr:nr + nvox], s * yy[nr + nvox:nr + 2 * nvox], s * yy[nr + 2 * nvox:])

        rhs = np.concatenate([b, np.zeros(3 * nvox)])
        rhs_norm = float(np.linalg.norm(rhs))
        starts.append(k)
        mon.have_prev = False
        if not warm:
            x = np.zeros(nvox)
        r = rhs.copy()
        if warm:
            r -= sf(x)
        s = sb(r)
        p = s.copy()
        gamma = float(s @ s)
        for _ in range(inner):
            if not gamma > 0:
                break
            q = sf(p)
            delta = float(q @ q)
            if not delta > 0:
                break
            alpha = gamma / delta
            x = x + alpha * p
            r = r - alpha * q
            k += 1
            if mon.record(k, x, float(np.linalg.norm(r)) / rhs_norm, lam):
                stopped = True
                break
            s = sb(r)
            gnew = float(s @ s)
            beta = gnew / gamma
            gamma = gnew
            p = s + beta * p
    return mon.result(x, k, outer_starts=np.array(starts))


def adjoint_discrepancy(fwd, back, nd, nr, trials, seed, dtype=np.float64):
    """tests/oracles.hpp:66-87 (N(0,1) trials; rng differs from mt19937_64, statistic is the same)."""
    rng = np.random.default_rng(seed)
    worst = 0.0
    for _ in range(trials):
        x = rng.standard_normal(nd).astype(dtype)
        y = rng.standard_normal(nr).astype(dtype)
        ax = fwd(x).astype(np.float64)
        by = back(y).astype(np.float64)
        lhs = float(ax @ y.astype(np.float64))
        rhs = float(x.astype(np.float64) @ by)
        sc = float(np.linalg.norm(ax) * np.linalg.norm(y.astype(np.float64)))
        if sc > 0:
            worst = max(worst, abs(lhs - rhs) / sc)
    return worst


def ray_box_chord(origin, d, lo, hi):
    """tests/oracles.hpp:89-107 (slab method)."""
    tmin, tmax = -math.inf, math.inf
    for a in range(3):
        if d[a] == 0.0:
            if origin[a] < lo[a] or origin[a] > hi[a]:
                return 0.0
            continue
        t1 = (lo[a] - origin[a]) / d[a]
        t2 = (hi[a] - origin[a]) / d[a]
        if t1 > t2:
            t1, t2 = t2, t1
        tmin, tmax = max(tmin, t1), min(tmax, t2)
    return max(0.0, tmax - tmin)
