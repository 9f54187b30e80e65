"""Band-sharded range of z-slab sharding on the CPU: the row partition
(ctk_band_partition, bands.cpp) -- the owned rows partition the detector, every slab's
rays stay inside its reached rows (checked with the oracle's forward of slab-only volumes),
and the held windows are a fraction of the detector at the C5 shape."""
import numpy as np
import pytest

from geoms import cone_bench, parallel3d, to_ctk


def _slabs(nz, world):
    from paper_2211_14212_b200.comm import shard_slabs

    return [shard_slabs(nz, world, r) for r in range(world)]


@pytest.mark.parametrize("world", [1, 2, 3, 5])
@pytest.mark.parametrize("name", ["cone", "parallel3d"])
def test_band_partition_contains_the_slab_rays(restated, name, world):
    import paper_2211_14212_b200 as ctk

    g = cone_bench(20, 12) if name == "cone" else parallel3d(nz=20)
    cg = to_ctk(g)
    sl = _slabs(g.nz, world)
    t0, t1, o0, o1 = ctk.band_partition(cg, [a for a, _ in sl], [b for _, b in sl])
    assert o0[0] == 0 and o1[-1] == g.nv
    for r in range(world):
        assert o0[r] <= o1[r] and (r == 0 or o0[r] == o1[r - 1])
    rng = np.random.default_rng(1)
    n = g.nx * g.ny
    for r, (z0, cnt) in enumerate(sl):
        x = np.zeros(g.domain_size)
        x[z0 * n:(z0 + cnt) * n] = rng.random(cnt * n) + 0.1
        y = restated.forward(g, x).reshape(len(g.angles), g.nv, g.nu)
        rows = np.nonzero(np.abs(y).sum(axis=(0, 2)))[0]
        if rows.size == 0:  # a slab outside the detector's field of view
            continue
        assert rows.min() >= t0[r] and rows.max() < t1[r], (r, rows.min(), rows.max(), t0[r], t1[r])


def test_band_windows_at_c5_shape():
    import paper_2211_14212_b200 as ctk

    g = ctk.ConeGeometry(ctk.BeamMode.cone3d, 2048.0, 1024.0, 1.5, 1024, 1024, ctk.VolumeShape(1024, 1024, 1024, 1.0),
                         [0.0])
    sl = _slabs(1024, 8)
    t0, t1, o0, o1 = ctk.band_partition(g, [a for a, _ in sl], [b for _, b in sl])
    held = [max(t1[r], o1[r]) - min(t0[r], o0[r]) for r in range(8)]
    assert max(held) <= 0.35 * 1024, held  # each rank holds about a third of the rows or less
    assert [o1[r] - o0[r] for r in range(8)] == [128] * 8


def test_band_partition_errors():
    import paper_2211_14212_b200 as ctk

    g = to_ctk(cone_bench(16, 4))
    with pytest.raises(ctk.ParameterError, match="tile z"):
        ctk.band_partition(g, [0, 9], [8, 8])
    with pytest.raises(ctk.ParameterError, match="cover the volume"):
        ctk.band_partition(g, [0, 8], [8, 4])
