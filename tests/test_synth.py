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


def test_cosine_modes_builder():
    """The blocked fp32 builder equals the fp64 outer-product definition (input generator only)."""
    shape = (3, 37, 29)
    modes = [(2, 5, 1), (0, 0, 2), (7, 0, 0)]
    amps = [0.1, -0.2, 0.05]
    a = synth.cosine_modes(shape, modes, amps, 0.3, block=8)
    z, y, x = np.meshgrid(np.arange(3), np.arange(37), np.arange(29), indexing="ij")
    ref = 0.3 + sum(am * synth.cosine_mode(x, k, 29) * synth.cosine_mode(y, l, 37) * synth.cosine_mode(z, m, 3)
                    for am, (k, l, m) in zip(amps, modes))
    assert np.array_equal(a, ref.astype(np.float32))
