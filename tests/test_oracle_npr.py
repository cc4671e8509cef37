"""Pins of the NEXT-1 oracle (the §6 NPR filter) against things other than
itself: SPEC's worked scale factor (golden), the filter's limit cases, and the dense minimiser
of the paper's energy evaluated link by link (oracle/brute.py)."""
import json
import os

import numpy as np
import pytest

import oracle as O
from oracle import brute

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "npr_spec.json")))


def _single_link_volume(diff):
    """3 x 3 x 3 zeros with one x-link of value `diff` at the centre voxel (its only
    non-zero forward difference)."""
    I = np.zeros((3, 3, 3))
    I[1, 1, 2] = diff
    return I


def test_scale_factor_at_sigma_and_saturation():
    s = GOLD["sigma_gray"] / 255.0
    lam = GOLD["lambda"]
    V = O.npr_gradient_field(_single_link_volume(s), lam, s)
    assert V["x"][1, 1, 1] / s == pytest.approx(GOLD["factor_at_sigma"], abs=1e-6)  # SPEC prints 6 digits
    big = GOLD["saturation_magnitude_gray"] / 255.0
    V = O.npr_gradient_field(_single_link_volume(big), lam, s)
    assert V["x"][1, 1, 1] / big == pytest.approx(GOLD["saturation_factor"], abs=1e-6)


def test_zero_gradient_and_constant_volume():
    I = np.full((4, 5, 6), 0.3)
    V = O.npr_gradient_field(I, 1.25, 5 / 255)
    assert all(np.all(v == 0) for v in V.values())
    x = O.npr_filter(I, alpha=0.001)
    assert np.abs(x - 0.3).max() < 1e-12


def test_identity_filter():
    """lambda = 1, sigma -> 0: V = grad I0, the energy's minimiser is I0 itself."""
    rng = np.random.default_rng(3)
    I = rng.random((5, 6, 7))
    x = O.npr_filter(I, alpha=0.001, lam=1.0, sigma=1e-9)
    assert np.abs(x - I).max() < 1e-8


@pytest.mark.parametrize("W,alpha", [((1.0, 1.0, 0.1), 0.001), ((0.5, 2.0, 1.0), 0.2)])
def test_matches_brute_force_energy_minimiser(W, alpha):
    rng = np.random.default_rng(7)
    shape = (2, 3, 4)
    I = rng.random(shape) * 0.2
    lam, sigma = 1.25, 0.05
    A, b = brute.quadratic_form(shape, W, alpha, V=I, G=brute.npr_G(I, lam, sigma))
    xb = brute.minimiser(A, b).reshape(shape)
    x = O.npr_filter(I, W=W, alpha=alpha, lam=lam, sigma=sigma, tol=1e-13)
    assert np.abs(x - xb).max() < 1e-9
    # and the assembled rhs is the energy's linear term
    assert np.abs(O.rhs_npr(I, W, alpha, lam, sigma).ravel() - b).max() < 1e-12


def test_suppresses_small_gradients():
    """Noise well below sigma is damped, a step far above sigma survives:
    the gradient energy across y (the step runs along x) drops by >= 4x, the step stays."""
    rng = np.random.default_rng(11)
    shape = (6, 24, 24)
    step = np.zeros(shape)
    step[:, :, 12:] = 0.5
    noisy = step + rng.normal(0, 0.002, shape)
    x = O.npr_filter(noisy, alpha=0.001, lam=1.25, sigma=5 / 255)
    rough = lambda u: np.mean(np.diff(u, axis=1) ** 2)
    assert rough(x) <= 0.25 * rough(noisy)
    jump = x[:, :, 14].mean() - x[:, :, 9].mean()
    assert 0.45 <= jump <= 0.70  # the step survives (lambda = 1.25 amplifies it a little)
