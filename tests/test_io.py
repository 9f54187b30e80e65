"""Raw f32 + .hdr I/O and the 16-bit PGM preview against the reference's src/io.cpp
(compiled unmodified into oracle/_ref/libctkref.so): byte-identical files both ways and the
same error classes."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle.oracle import Reference

pytestmark = pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def ref():
    return Reference().lib


@pytest.fixture(scope="module")
def io():
    from paper_2211_14212_b200 import io as m

    return m


def _fp(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def test_volume_roundtrip_byte_identical(ref, io, tmp_path):
    import paper_2211_14212_b200 as ctk

    rng = np.random.default_rng(1)
    shape = ctk.VolumeShape(5, 4, 3, 0.7)
    x = rng.standard_normal(shape.size()).astype(np.float32)
    ours, theirs = str(tmp_path / "ours.raw"), str(tmp_path / "theirs.raw")
    io.save_volume(ours, x, shape)
    assert ref.ref_save_volume(theirs.encode(), 5, 4, 3, C.c_double(0.7), _fp(x, C.c_float)) == 0
    for suffix in ("", ".hdr"):
        assert open(ours + suffix, "rb").read() == open(theirs + suffix, "rb").read()
    data, sh = io.load_volume(theirs)
    assert np.array_equal(data, x) and (sh.nx, sh.ny, sh.nz, sh.spacing) == (5, 4, 3, 0.7)
    dims = (C.c_int * 3)()
    sp = C.c_double()
    back = np.zeros_like(x)
    assert ref.ref_load_volume(ours.encode(), dims, C.byref(sp), _fp(back, C.c_float), C.c_size_t(back.size)) == 0
    assert list(dims) == [5, 4, 3] and sp.value == 0.7 and np.array_equal(back, x)


def test_projections_roundtrip_byte_identical(ref, io, tmp_path):
    import paper_2211_14212_b200 as ctk

    rng = np.random.default_rng(2)
    angles = np.array(ctk.equidistant_angles(7))
    y = rng.standard_normal(7 * 3 * 4).astype(np.float32)
    ours, theirs = str(tmp_path / "p_ours.raw"), str(tmp_path / "p_theirs.raw")
    io.save_projections(ours, y, angles, 4, 3)
    assert ref.ref_save_projections(theirs.encode(), 7, 4, 3, _fp(angles, C.c_double), _fp(y, C.c_float)) == 0
    for suffix in ("", ".hdr"):
        assert open(ours + suffix, "rb").read() == open(theirs + suffix, "rb").read()
    data, ang, nu, nv = io.load_projections(theirs)
    assert np.array_equal(data, y) and ang == list(angles) and (nu, nv) == (4, 3)


def test_pgm16_byte_identical(ref, io, tmp_path):
    rng = np.random.default_rng(3)
    v = (rng.standard_normal(6 * 5) * 2.0).astype(np.float32)
    for wmin, wmax in ((-1.0, 1.5), (0.0, 0.0), (-3.0, 3.0)):
        ours, theirs = str(tmp_path / "o.pgm"), str(tmp_path / "t.pgm")
        io.write_pgm16(ours, 6, 5, v, wmin, wmax)
        assert ref.ref_write_pgm16(theirs.encode(), 6, 5, _fp(v, C.c_float), C.c_double(wmin), C.c_double(wmax)) == 0
        assert open(ours, "rb").read() == open(theirs, "rb").read()


def test_io_errors_match(ref, io, tmp_path):
    import paper_2211_14212_b200 as ctk

    missing = str(tmp_path / "nope.raw")
    with pytest.raises(ctk.ParameterError):
        io.load_volume(missing)
    dims = (C.c_int * 3)()
    sp = C.c_double()
    assert ref.ref_load_volume(missing.encode(), dims, C.byref(sp), None, C.c_size_t(0)) == 3  # ParameterError
    # a raw file shorter than its header promises -> DimensionError on both sides
    short = str(tmp_path / "short.raw")
    io.save_volume(short, np.zeros(8, np.float32), ctk.VolumeShape(2, 2, 2, 1.0))
    with open(short, "wb") as f:
        f.write(b"\0" * 12)
    with pytest.raises(ctk.DimensionError):
        io.load_volume(short)
    assert ref.ref_load_volume(short.encode(), dims, C.byref(sp), None, C.c_size_t(0)) == 1
    with open(short + ".hdr", "w") as h:
        h.write("2 2\n")
    with pytest.raises(ctk.ParameterError):
        io.load_volume(short)
    assert ref.ref_load_volume(short.encode(), dims, C.byref(sp), None, C.c_size_t(0)) == 3
    with pytest.raises(ctk.DimensionError):
        io.write_pgm16(str(tmp_path / "x.pgm"), 0, 3, np.zeros(3, np.float32), 0.0, 1.0)
