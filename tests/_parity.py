"""Shared checks of the GPU parity tests (test helpers, no method arithmetic)."""
import numpy as np

DELTA = 1e-6  # AMB-9 multiplet guard (the library default, tdvp_params.multiplet_delta)


def check_spectra(a, b, eps, tol, weight_tol=None):
    """Compare one bond's spectra, a (GPU) and b (oracle), both descending.

    The common prefix must agree to tol * sigma_1.  Values kept by one side
    only must be eps-threshold or multiplet-guard flips (DESIGN.md R-F, R-9b):
    within the cut's uncertainty band of eps * sigma_1, or continuing a
    multiplet (gap <= DELTA * sigma + band) from the last common value.  The
    band is 4x the measured GPU-oracle difference of the common spectrum at
    this bond, floor 1e-13 sigma_1 (the SVDs' own rounding for n <= 2048).

    weight_tol (long truncated runs, DESIGN.md R-F2): a value that flipped at
    the cut in an earlier step keeps evolving on the side that kept it, so
    after a few steps one side may hold a short tail that is no longer at the
    cut.  Such a tail is accepted when its total weight sqrt(sum x^2) is at
    most weight_tol * sigma_1, i.e. it accounts for a state difference below
    that tolerance (the eps rule itself is pinned exactly by the SVD tests).
    Returns |chi_gpu - chi_oracle|."""
    k = min(len(a), len(b))
    s1 = b[0]
    dpre = float(np.abs(np.asarray(a[:k]) - np.asarray(b[:k])).max())
    assert dpre <= tol * s1, (len(a), len(b), dpre / s1)
    band = max(4.0 * dpre, 1e-13 * s1)
    longer = a if len(a) > len(b) else b
    tail = np.asarray(longer[k:])
    if weight_tol is not None and len(tail) and float(np.sqrt(np.sum(tail ** 2))) <= weight_tol * s1:
        return abs(len(a) - len(b))
    prev = longer[k - 1]
    for x in tail:
        at_eps = abs(x - eps * s1) <= band
        in_multiplet = prev - x <= DELTA * prev + band
        assert at_eps or in_multiplet, (len(a), len(b), x / s1, prev / s1, band / s1)
        prev = x
    return abs(len(a) - len(b))
