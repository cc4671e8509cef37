"""The shared seeded generator (gdp_synth): deterministic, per-slice keyed, right ranges."""
import numpy as np

import gdp_synth as synth


def test_deterministic_and_per_slice_keyed():
    a = synth.make_stack(40, 30, 4, 7, "u8")
    b = synth.make_stack(40, 30, 6, 7, "u8")
    assert np.array_equal(a, b[:4])  # slice z depends only on (seed, z)
    c = synth.make_stack(40, 30, 4, 8, "u8")
    assert not np.array_equal(a, c)


def test_ranges_and_dtypes():
    f = synth.make_stack(64, 64, 3, 0, "f32")
    assert f.dtype == np.float32 and f.min() >= 0.0 and f.max() <= 1.0
    u = synth.make_stack(64, 64, 3, 0, "u8")
    assert u.dtype == np.uint8
    s = synth.make_slice(64, 64, 0, 1)
    assert np.array_equal(u[1], np.rint(255.0 * s).astype(np.uint8))


def test_offset_striped_no_clipping():
    I0, T, c = synth.offset_striped_u8(50, 40, 12, 1)
    assert T.min() >= 20 and T.max() <= 235 and np.abs(c).max() <= 20
    assert np.array_equal(I0.astype(np.int32), T[None] + c[:, None, None])
