"""Buffer checks of the operator entry points (no GPU needed: they fire before any native
call): mixed host/device operands, mismatched dtypes and non-contiguous outputs are
rejected instead of being read or written as flat arrays."""
import numpy as np
import pytest


def test_projector_buffer_checks():
    import paper_2211_14212_b200 as ctk
    from paper_2211_14212_b200.api import Projector

    a = np.zeros(8, np.float32)
    with pytest.raises(ctk.ParameterError, match="dtypes differ"):
        Projector._check_buffers(a, np.zeros(8, np.float64))
    with pytest.raises(ctk.ParameterError, match="contiguous"):
        Projector._check_buffers(a, np.zeros(16, np.float32)[::2])
    with pytest.raises(ctk.ParameterError, match="contiguous"):
        Projector._check_buffers(np.zeros(8, ">f4"), np.zeros(8, ">f4"))
    Projector._check_buffers(a, np.zeros(3, np.float32))  # sizes are checked by the callers


def test_contiguous_inputs_are_normalised():
    from paper_2211_14212_b200.api import _contiguous

    x = np.arange(16, dtype=np.float32)[::2]
    c = _contiguous(x)
    assert c.flags.c_contiguous and np.array_equal(c, x)
    b = _contiguous(np.arange(4, dtype=">f8"))
    assert b.dtype.isnative and np.array_equal(b, [0, 1, 2, 3])
    assert _contiguous([1.0, 2.0]).dtype == np.float64
