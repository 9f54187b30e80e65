"""Separate handles may run concurrently (SURVEY.md 8(b) threading contract; the reference's
operator applications are pure): four host threads, each with its own
projector pair (different geometries and precisions), run forward / back projections and
an LSQR solve at the same time; every result must equal the one computed alone, bitwise."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _work(ctk, n, na, dtype, variant):
    g = ctk.bench_geometry(n, na)
    pair = ctk.projector_pair(g, variant, dtype=dtype)
    x = np.random.default_rng(n + na).random(pair.domain_size).astype(dtype)
    y = pair.apply_forward(x)
    bt = pair.apply_back(y)
    r = ctk.lsqr(pair, y, ctk.SolverOptions(max_iters=4, residual_tolerance=0.0,
                                            stop_on_explicit_residual_increase=False))
    return y, bt, np.asarray(r.x), list(r.log.explicit_residual)


def test_concurrent_handles_bitwise():
    import paper_2211_14212_b200 as ctk

    jobs = [(40, 30, np.float32, ctk.BackprojectVariant.matched),
            (48, 24, np.float32, ctk.BackprojectVariant.voxel_driven),
            (32, 20, np.float64, ctk.BackprojectVariant.matched),
            (56, 36, np.float32, ctk.BackprojectVariant.matched)]
    alone = [_work(ctk, *j) for j in jobs]
    out = [None] * len(jobs)
    errs = []

    def run(i):
        try:
            for _ in range(3):
                out[i] = _work(ctk, *jobs[i])
        except Exception as e:  # surfaced below
            errs.append(e)

    ts = [threading.Thread(target=run, args=(i,)) for i in range(len(jobs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for a, b in zip(alone, out):
        for u, v in zip(a[:3], b[:3]):
            assert np.array_equal(u, v)
        assert a[3] == b[3]
