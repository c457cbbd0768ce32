"""Pins of the oracle's temporal MB-importance reuse against things
other than itself: SPEC's worked examples (restated; S:135-137 Phi, S:145-147 series,
S:154-156 CDF pick, S:162-164 budget), scipy's connected-component labelling + exact rational sums
(fractions.Fraction) for Phi, a direct CDF walk, and invariants. CPU only."""
from fractions import Fraction

import numpy as np
import pytest
import scipy.ndimage as ndi

import oracle
import synth


def _exact_phi(mask: np.ndarray) -> tuple[float, int]:
    """Sum of the correctly rounded fp64 terms 1.0/area over scipy's 4-connected components, summed
    exactly (Fraction) and rounded once (reading D18)."""
    lab, n = ndi.label(mask, structure=ndi.generate_binary_structure(2, 1))
    areas = np.bincount(lab.reshape(-1))[1:]
    return float(sum((Fraction(1.0 / float(a)) for a in areas), Fraction(0))), int(n)


def test_phi_spec_examples():
    z = np.zeros((16, 16), np.int16)
    assert oracle.phi_inv_area(z, 0) == (0.0, 0)                        # S:135 all-zero -> 0
    r = z.copy()
    r[5:7, 5:7] = 20
    assert oracle.phi_inv_area(r, 8) == (0.25, 1)                      # S:136 one 2x2 block -> 1/4
    r = z.copy()
    r[0, 0] = -9                                                        # negative residuals count (|r|)
    r[8:11, 8:11] = 30                                                  # areas 1 and 9
    phi, n = oracle.phi_inv_area(r, 8)
    assert n == 2 and phi == float(Fraction(1) + Fraction(1.0 / 9.0))  # S:137 -> 1 + 1/9
    assert oracle.phi_inv_area(r, 9)[1] == 1                           # foreground is |r| > thr (strict)


@pytest.mark.parametrize("seed,p", [(0, 0.3), (1, 0.5), (2, 0.62), (3, 0.05)])
def test_phi_matches_scipy_components_and_exact_sum(seed, p):
    rng = np.random.default_rng(seed)
    r = (rng.random((57, 83)) < p).astype(np.int16) * rng.integers(-50, 51, size=(57, 83)).astype(np.int16)
    phi, n = oracle.phi_inv_area(r, 7)
    ref, nref = _exact_phi(np.abs(r) > 7)
    assert n == nref and phi == ref


def test_phi_on_synthetic_residuals_is_the_exact_sum():
    res = synth.residuals_y(1, 3, 180, 320, 4)
    for f in range(3):
        phi, n = oracle.phi_inv_area(res[0, f], 8)
        ref, nref = _exact_phi(np.abs(res[0, f].astype(np.int32)) > 8)
        assert (phi, n) == (ref, nref)


def test_delta_series_spec_examples():
    a, T, S, M = oracle.delta_series([1.0, 2.0, 3.0, 4.0])
    assert a == [1.0, 1.0, 1.0] and S == [1 / 3, 1 / 3, 1 / 3]
    a, T, S, M = oracle.delta_series([5.0, 5.0, 5.0])                    # S:146 degenerate
    assert T == 0.0 and S == [0.0, 0.0] and M == [0.0, 0.0, 0.0]
    a, T, S, M = oracle.delta_series([0.0, 4.0, 1.0])                    # S:147 |dPhi| = {4, 3}
    assert S == [4 / 7, 3 / 7] and M == [0.0, 4 / 7, 4 / 7 + 3 / 7]


def test_cdf_pick_spec_examples():
    F = 30
    _, _, _, M = oracle.delta_series([float(i) for i in range(F)])       # uniform mass
    assert oracle.cdf_pick(M, 30, F) == list(range(F))                   # S:154 full budget: every frame
    j = 17
    phi = [0.0] * j + [5.0] * (F - j)                                    # all mass on the change into frame j
    _, _, _, M = oracle.delta_series(phi)
    assert oracle.cdf_pick(M, 5, F) == [0, j]                            # S:155 point mass collapses
    # normalized {.1,.1,.1,.1,.6} over a 6-frame chunk, 3 intervals -> direct CDF walk
    phi = [0.0, 1.0, 2.0, 3.0, 4.0, 10.0]
    _, _, S, M = oracle.delta_series(phi)
    assert S == pytest.approx([0.1, 0.1, 0.1, 0.1, 0.6])
    cdf = np.cumsum([0.0] + S)                                           # cdf[k] = sum_{i<k} S_i
    walk = [0] + [int(np.flatnonzero(cdf[1:] >= (t + 0.5) / 3)[0]) + 1 for t in range(3)]
    assert oracle.cdf_pick(M, 4, 6) == sorted(set(walk)) == [0, 2, 5]


def test_allocate_budget_spec_examples():
    assert oracle.allocate_budget([3.0, 1.0], 8, 30) == [6, 2]            # S:162 exact proportionality
    assert oracle.allocate_budget([1.0, 1.0], 5, 30) == [3, 2]            # S:163 tie -> lower stream
    assert oracle.allocate_budget([2.5], 7, 30) == [7]                   # S:164 one stream
    assert oracle.allocate_budget([0.0, 0.0, 0.0], 7, 30) == [3, 2, 2]    # no change anywhere: even split
    assert oracle.allocate_budget([1.0, 5.0], 100, 30) == [11, 30]       # capped at F frames (not redistributed)
    assert oracle.allocate_budget([1.0, 2.0], 1, 30) == [1, 1]           # every stream keeps its anchor


@pytest.mark.parametrize("budget", [2, 9, 40, 200])
def test_temporal_select_invariants(budget):
    res = synth.residuals_y(3, 30, 90, 160, 5)
    o = oracle.temporal_select(res, 8, budget)
    n = o["frames_per_stream"]
    assert n.sum() <= max(budget, 3) and (n >= 1).all() and (n <= 30).all()
    for s in range(3):
        sel = np.flatnonzero(o["selected"][s])
        assert sel[0] == 0 and len(sel) <= n[s]
        ru = o["reuse"][s]
        assert (o["selected"][s][ru] == 1).all() and (ru <= np.arange(30)).all()
        assert (ru[sel] == sel).all()                                     # selected frames reuse themselves
        for f in range(30):
            assert ru[f] == sel[sel <= f].max()                           # the nearest selected frame before
