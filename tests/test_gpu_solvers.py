"""Device-resident solvers vs the reference solvers (oracle/_ref, T=double golden).

Bars (north_star): iterates after k iterations within 1e-4 relative L2, and the residual
history within 1e-4 per iteration.  Also: bitwise rerun determinism
(test_solvers.cpp:436-451) and the error taxonomy.
"""
import numpy as np
import pytest

from geoms import cone_bench, cone_default, parallel2d, to_ctk
from conftest import rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def ctk():
    import paper_2211_14212_b200 as m

    m.load()
    return m


@pytest.fixture(scope="module")
def problem(restated, reference):
    g = cone_bench(32, 40)
    gt = restated.shepp_logan_3d(32, np.float64)
    b = reference.forward(g, gt)
    return g, gt, b


def _opts(ctk, k, gt=None):
    return ctk.SolverOptions(max_iters=k, stop_on_explicit_residual_increase=False, residual_tolerance=0.0,
                             ground_truth=gt)


def _check_hist(res, want):
    impl = np.array(res.log.implicit_residual)
    expl = np.array(res.log.explicit_residual)
    assert res.iterations_run == want["iterations_run"]
    assert np.all(np.abs(expl - want["explicit"]) <= TOL * np.abs(want["explicit"]))
    assert np.all(np.abs(impl - want["implicit"]) <= TOL * np.abs(want["implicit"]))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("solver", ["cgls", "lsqr", "lsmr"])
def test_solver_parity(ctk, reference, problem, dtype, solver):
    g, gt, b = problem
    k = 12
    lam = 30.0 if solver == "lsmr" else 0.0
    reference.set_threads(8)
    try:
        want = reference.solve(g, b, solver, k, lam=lam, tol=0.0, stop_inc=False, gt=gt)
    finally:
        reference.set_threads(1)
    pair = ctk.projector_pair(to_ctk(g), dtype=dtype)
    opts = _opts(ctk, k, gt.astype(dtype))
    if solver == "lsmr":
        res = ctk.lsmr(pair, b.astype(dtype), lam, opts)
    else:
        res = getattr(ctk, solver)(pair, b.astype(dtype), opts)
    assert rel_l2(res.x, want["x"]) < TOL
    _check_hist(res, want)
    err = np.array(res.log.relative_error)
    assert np.all(np.abs(err - want["relative_error"]) <= TOL * want["relative_error"])
    if solver == "lsmr":
        assert res.log.lambda_ == [lam] * k


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_hybrid_lsqr_gcv_parity(ctk, reference, problem, dtype):
    g, gt, b = problem
    k = 8
    want = reference.solve(g, b, "hybrid_lsqr", k, strategy=2, tol=0.0, stop_inc=False)
    pair = ctk.projector_pair(to_ctk(g), dtype=dtype)
    res = ctk.hybrid_lsqr(pair, b.astype(dtype), ctk.HybridStrategy.gcv(), _opts(ctk, k))
    assert rel_l2(res.x, want["x"]) < TOL
    _check_hist(res, want)
    assert np.allclose(res.log.lambda_, want["lambda"], rtol=1e-3)
    assert res.stored_domain_basis == want["stored_domain_basis"]
    assert res.stored_range_basis == want["stored_range_basis"]


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_cgls_tv_parity(ctk, reference, problem, dtype):
    g, gt, b = problem
    outer, inner, lam = 2, 4, 0.5
    want = reference.solve(g, b, "cgls_tv", 1, lam=lam, outer=outer, inner=inner, tol=0.0, stop_inc=False)
    pair = ctk.projector_pair(to_ctk(g), dtype=dtype)
    res = ctk.cgls_tv(pair, b.astype(dtype), lam, outer, inner, _opts(ctk, 1))
    assert rel_l2(res.x, want["x"]) < TOL
    _check_hist(res, want)
    assert list(res.outer_starts) == list(want["outer_starts"])


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_sirt_parity(ctk, reference, problem, dtype):
    g, gt, b = problem
    k = 10
    want = reference.solve(g, b, "sirt", k, tol=0.0, stop_inc=False, gt=gt)
    pair = ctk.projector_pair(to_ctk(g), dtype=dtype)
    res = ctk.sirt(pair, b.astype(dtype), _opts(ctk, k, gt.astype(dtype)))
    assert rel_l2(res.x, want["x"]) < TOL
    _check_hist(res, want)
    assert res.log.lambda_ == []
    z = ctk.sirt(pair, np.zeros_like(b, dtype=dtype), _opts(ctk, k))
    assert z.iterations_run == 0 and z.stop_reason.name == "tolerance" and not np.any(z.x)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("variant", ["ab_gmres", "ba_gmres"])
def test_gmres_parity(ctk, reference, problem, dtype, variant):
    g, gt, b = problem
    k = 8
    want = reference.solve(g, b, variant, k, tol=0.0, stop_inc=False, gt=gt)
    pair = ctk.projector_pair(to_ctk(g), dtype=dtype)
    res = getattr(ctk, variant)(pair, b.astype(dtype), _opts(ctk, k, gt.astype(dtype)))
    assert rel_l2(res.x, want["x"]) < TOL
    _check_hist(res, want)
    assert res.stored_domain_basis == want["stored_domain_basis"]
    assert res.stored_range_basis == want["stored_range_basis"]


# fixed lambda: compared at k = 3 (the reference algorithm amplifies rounding-level
# perturbations ~30x per iteration there; see test_oracle.py / DESIGN.md)
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("strategy,k", [("gcv", 6), ("fixed", 3)])
def test_flsqr_tv_parity(ctk, reference, problem, dtype, strategy, k):
    g, gt, b = problem
    sid = {"fixed": 0, "gcv": 2}[strategy]
    want = reference.solve(g, b, "flsqr_tv", k, strategy=sid, lam=5.0, tol=0.0, stop_inc=False, gt=gt)
    pair = ctk.projector_pair(to_ctk(g), dtype=dtype)
    st = ctk.HybridStrategy.gcv() if strategy == "gcv" else ctk.HybridStrategy.fixed(5.0)
    res = ctk.flsqr_tv(pair, b.astype(dtype), st, _opts(ctk, k, gt.astype(dtype)))
    assert rel_l2(res.x, want["x"]) < TOL
    _check_hist(res, want)
    assert np.allclose(res.log.lambda_, want["lambda"], rtol=1e-3)
    assert [int(w.rsplit(" ", 1)[1]) for w in res.warnings] == list(want["warning_iterations"])
    assert res.stored_domain_basis == want["stored_domain_basis"]
    assert res.stored_range_basis == want["stored_range_basis"]
    with pytest.raises(ctk.ParameterError):
        ctk.flsqr_tv(pair, b.astype(dtype), ctk.HybridStrategy.dp(0.01), _opts(ctk, k))


def test_voxel_driven_lsqr_parity(ctk, reference, problem):
    g, gt, b = problem
    k = 6
    want = reference.solve(g, b, "lsqr", k, variant=1, tol=0.0, stop_inc=False)
    pair = ctk.projector_pair(to_ctk(g), ctk.BackprojectVariant.voxel_driven, dtype=np.float64)
    res = ctk.lsqr(pair, b, _opts(ctk, k))
    assert rel_l2(res.x, want["x"]) < TOL
    _check_hist(res, want)


@pytest.mark.parametrize("solver", ["cgls", "lsqr", "lsmr", "sirt", "hybrid_lsqr", "ab_gmres", "ba_gmres", "cgls_tv"])
@pytest.mark.parametrize("variant,tol", [(1, 1e-6), (0, 0.05)])
def test_stopping_rules_match(ctk, reference, solver, variant, tol):
    """The reference's stopping rules (solve_log.hpp:129-137): on a noisy unmatched run the
    explicit-residual-increase stop, on a matched run a residual tolerance -- same stop
    reason at the same iteration."""
    g = parallel2d(32, 30)
    rng = np.random.default_rng(3)
    x = rng.random(g.domain_size)
    b = reference.forward(g, x) + (0.05 if variant == 1 else 0.01) * rng.standard_normal(g.range_size)
    want = reference.solve(g, b, solver, 60, variant=variant, lam=0.5, strategy=2 if solver == "hybrid_lsqr" else 0,
                           outer=3, inner=20, tol=tol)
    pair = ctk.projector_pair(to_ctk(g), ctk.BackprojectVariant(variant), dtype=np.float64)
    opts = ctk.SolverOptions(max_iters=60, residual_tolerance=tol)
    if solver == "lsmr":
        res = ctk.lsmr(pair, b, 0.5, opts)
    elif solver == "hybrid_lsqr":
        res = ctk.hybrid_lsqr(pair, b, ctk.HybridStrategy.gcv(), opts)
    elif solver == "cgls_tv":
        res = ctk.cgls_tv(pair, b, 0.5, 3, 20, opts)
    else:
        res = getattr(ctk, solver)(pair, b, opts)
    assert res.stop_reason.name == want["stop_reason"]
    assert res.iterations_run == want["iterations_run"]


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_determinism_bitwise(ctk, problem, dtype):
    g, gt, b = problem
    pair = ctk.projector_pair(to_ctk(g), dtype=dtype)
    opts = ctk.SolverOptions(max_iters=6, ground_truth=gt.astype(dtype))
    r1 = ctk.lsqr(pair, b.astype(dtype), opts)
    r2 = ctk.lsqr(pair, b.astype(dtype), opts)
    assert r1.log.implicit_residual == r2.log.implicit_residual
    assert r1.log.explicit_residual == r2.log.explicit_residual
    assert r1.log.relative_error == r2.log.relative_error
    assert np.array_equal(r1.x, r2.x)


def test_device_resident_matches_host_entry(ctk, problem):
    import torch

    g, gt, b = problem
    pair = ctk.projector_pair(to_ctk(g))
    opts = _opts(ctk, 5)
    rh = ctk.lsmr(pair, b.astype(np.float32), 30.0, opts)
    rd = ctk.lsmr(pair, torch.from_numpy(b.astype(np.float32)).cuda(), 30.0, opts)
    assert np.array_equal(rd.x.cpu().numpy(), rh.x)
    assert rd.log.explicit_residual == rh.log.explicit_residual


def test_solver_errors(ctk):
    g = to_ctk(parallel2d(16, 8))
    pair = ctk.projector_pair(g, dtype=np.float64)
    with pytest.raises(ctk.DegenerateInputError):
        ctk.cgls(pair, np.zeros(pair.range_size), ctk.SolverOptions())
    with pytest.raises(ctk.ParameterError):
        ctk.cgls(pair, np.ones(pair.range_size), ctk.SolverOptions(max_iters=0))
    with pytest.raises(ctk.ParameterError):
        ctk.lsqr(pair, np.ones(pair.range_size), ctk.SolverOptions(residual_tolerance=-1.0))
    with pytest.raises(ctk.ParameterError):
        ctk.lsmr(pair, np.ones(pair.range_size), -0.5, ctk.SolverOptions())
    with pytest.raises(ctk.ParameterError):
        ctk.cgls_tv(pair, np.ones(pair.range_size), 0.0, 1, 1, ctk.SolverOptions())
    with pytest.raises(ctk.DimensionError):
        ctk.cgls(pair, np.ones(5), ctk.SolverOptions())


def test_observer_sees_iterates(ctk, problem):
    g, gt, b = problem
    pair = ctk.projector_pair(to_ctk(g))
    seen = []
    opts = _opts(ctk, 3)
    opts.iterate_observer = lambda k, x: seen.append((k, float(np.linalg.norm(x))))
    res = ctk.cgls(pair, b.astype(np.float32), opts)
    assert [k for k, _ in seen] == [1, 2, 3]
    assert abs(seen[-1][1] - np.linalg.norm(res.x)) < 1e-6 * np.linalg.norm(res.x)


def test_blas1_deterministic(ctk):
    import ctypes as C

    import torch

    lib = ctk.load()
    x = torch.randn(10_000_019, device="cuda", dtype=torch.float32)
    y = torch.randn(10_000_019, device="cuda", dtype=torch.float32)
    outs = []
    for _ in range(3):
        d = C.c_double()
        assert lib.ctk_dot_f32(x.numel(), C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), C.byref(d), None) == 0
        outs.append(d.value)
    assert outs[0] == outs[1] == outs[2]
    want = float((x.double() * y.double()).sum())
    assert abs(outs[0] - want) <= 1e-12 * abs(want) * 100 + 1e-9


@pytest.mark.parametrize("strategy", ["dp", "fixed"])
def test_hybrid_lsqr_dp_fixed_parity(ctk, reference, problem, strategy):
    g, gt, b = problem
    k = 8
    sid = {"fixed": 0, "dp": 1}[strategy]
    want = reference.solve(g, b, "hybrid_lsqr", k, strategy=sid, lam=0.5, noise_level=0.01, tol=0.0, stop_inc=False)
    pair = ctk.projector_pair(to_ctk(g), dtype=np.float64)
    st = ctk.HybridStrategy.fixed(0.5) if strategy == "fixed" else ctk.HybridStrategy.dp(0.01)
    res = ctk.hybrid_lsqr(pair, b, st, _opts(ctk, k))
    assert rel_l2(res.x, want["x"]) < TOL
    _check_hist(res, want)
    assert np.allclose(res.log.lambda_, want["lambda"], rtol=1e-3, atol=1e-12)


@pytest.mark.parametrize("solver", ["sirt", "ab_gmres", "ba_gmres", "cgls"])
def test_unmatched_pair_solver_parity(ctk, reference, problem, solver):
    """The voxel-driven (unmatched) backprojector through the newer solvers (f64)."""
    g, gt, b = problem
    k = 6
    want = reference.solve(g, b, solver, k, variant=1, tol=0.0, stop_inc=False)
    pair = ctk.projector_pair(to_ctk(g), ctk.BackprojectVariant.voxel_driven, dtype=np.float64)
    res = getattr(ctk, solver)(pair, b, _opts(ctk, k))
    assert rel_l2(res.x, want["x"]) < TOL
    _check_hist(res, want)


def test_cgls_tv_warm_start_parity(ctk, reference, problem):
    g, gt, b = problem
    outer, inner, lam = 2, 3, 0.5
    want = reference.solve(g, b, "cgls_tv", 1, lam=lam, outer=outer, inner=inner, warm=True, tol=0.0, stop_inc=False)
    pair = ctk.projector_pair(to_ctk(g), dtype=np.float64)
    res = ctk.cgls_tv(pair, b, lam, outer, inner, _opts(ctk, 1), warm_start=True)
    assert rel_l2(res.x, want["x"]) < TOL
    _check_hist(res, want)


def test_siddon_lsqr_matches_restated(ctk, restated):
    """Siddon has no reference implementation: the device LSQR on the Siddon pair against the
    numpy LSQR recurrence on the (pinned) C restatement of the same operators."""
    from geoms import cone_bench
    from oracle.oracle import lsqr as lsqr_np

    g = cone_bench(24, 20)
    gt = restated.shepp_logan_3d(24, np.float64)
    b = restated.siddon_forward(g, gt)
    want = lsqr_np(lambda v: restated.siddon_forward(g, v), lambda v: restated.siddon_back(g, v), b, 8, tol=0.0,
                   stop_inc=False)
    pair = ctk.projector_pair(to_ctk(g), dtype=np.float64, projector=ctk.ProjectorKind.siddon)
    res = ctk.lsqr(pair, b, _opts(ctk, 8))
    assert rel_l2(res.x, want["x"]) < 1e-9
    assert np.allclose(res.log.explicit_residual, want["explicit"], rtol=1e-9)


@pytest.mark.parametrize("solver", ["cgls", "lsqr", "lsmr", "sirt", "hybrid_lsqr", "ab_gmres", "ba_gmres", "cgls_tv"])
@pytest.mark.parametrize("bad", ["inf", "nan", "zero"])
def test_error_behaviour_matches_reference(ctk, problem, reference, solver, bad):
    """Non-finite or zero measurements: the same error class (and, for a NumericalError, the
    same iteration) as the reference's solver (IterationMonitor::record's finite check,
    solve_log.hpp:116-117; the zero-b guards)."""
    from oracle.oracle import RefError

    g, gt, b = problem
    b = b.copy()
    if bad == "zero":
        b[:] = 0.0
    else:
        b[b.size // 3] = np.inf if bad == "inf" else np.nan
    codes = {1: ctk.DimensionError, 2: ctk.GeometryError, 3: ctk.ParameterError, 4: ctk.DegenerateInputError,
             5: ctk.NumericalError}
    try:
        reference.solve(g, b, solver, 5, lam=1.0, strategy=2 if solver == "hybrid_lsqr" else 0, outer=2, inner=3,
                        tol=0.0, stop_inc=False)
        want = None
    except RefError as e:
        want = e
    pair = ctk.projector_pair(to_ctk(g), dtype=np.float64)
    opts = _opts(ctk, 5)
    if solver == "lsmr":
        def run():
            return ctk.lsmr(pair, b, 1.0, opts)
    elif solver == "hybrid_lsqr":
        def run():
            return ctk.hybrid_lsqr(pair, b, ctk.HybridStrategy.gcv(), opts)
    elif solver == "cgls_tv":
        def run():
            return ctk.cgls_tv(pair, b, 1.0, 2, 3, opts)
    else:
        def run():
            return getattr(ctk, solver)(pair, b, opts)
    if want is None:
        run()
        return
    with pytest.raises(codes[want.code]) as e:
        run()
    if want.code == 5:
        assert e.value.iteration == want.iteration
