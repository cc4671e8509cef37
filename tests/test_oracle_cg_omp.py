"""Pins of the C/OpenMP CG oracle (oracle/cg_omp.c) — the CPU baseline bench.py times — against
the numpy oracle (itself pinned in test_oracle.py) and the DCT closed form."""
import numpy as np

import gdp_synth as synth
import oracle as O
from oracle import cg_omp


def test_c_oracle_matches_numpy_oracle_config0():
    I0 = synth.make_config(0)
    I1c = cg_omp.diffuse_z(I0)
    I1n = O.diffuse_z(I0)
    assert np.abs(I1c - I1n).max() < 1e-8
    I2c = cg_omp.screened_poisson_slices(I0, I1n, 0.01)
    I2n = O.screened_poisson_slices(I0, I1n, 0.01)
    assert np.abs(I2c - I2n).max() < 1e-8


def test_c_oracle_u8_ragged_matches_dct():
    I0 = synth.make_stack(45, 33, 7, 3, "u8")
    I1 = cg_omp.diffuse_z(I0, W=(1.0, 0.7, 0.25))
    assert np.abs(I1 - O.diffuse_z_dct(I0, W=(1.0, 0.7, 0.25))).max() < 1e-8
    assert abs(I1.mean() - O.decode(I0).mean()) < 1e-13  # mean pin (c-3)
    I2 = cg_omp.screened_poisson_slices(I0, I1, 0.1)
    assert np.abs(I2 - O.screened_poisson_slices_dct(I0, I1, 0.1)).max() < 1e-8


def test_c_oracle_closed_forms():
    I0u, T, c = synth.offset_striped_u8(20, 18, 9, 3)  # P6: I1 = I2 = T + mean(c)
    exp = (T[None].astype(np.float64) + c.mean()) / 255.0
    I1 = cg_omp.diffuse_z(I0u)
    assert np.abs(I1 - exp).max() < 1e-7
    assert np.abs(cg_omp.screened_poisson_slices(I0u, I1, 0.01) - exp).max() < 1e-7
    assert cg_omp.threads() >= 1
