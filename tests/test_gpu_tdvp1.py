"""GPU: serial one-site TDVP (tdvp_step1) and the hybrid 2TDVP -> 1TDVP step
(tdvp_step_hybrid) against the 1TDVP oracle
(oracle/tdvp1.py) on the same seeded inputs, plus the invariants 1TDVP keeps
on the device (energy, norm, bond dimensions)."""
import numpy as np
import pytest

import tdvp_inputs as ti
from oracle import tdvp as O
from oracle import tdvp1 as T1

from _parity import check_spectra

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1912_06127_b200 as pkg
    return pkg


def _pair(B, mps, W, chi_max, eps):
    D_ = max(max(w.shape[0], w.shape[3]) for w in W)
    t = B.Tdvp(len(W), 2, D_, chi_max)
    t.set_params(eps=eps)
    t.set_mpo(W)
    t.set_mps(mps.psi, mps.lam)
    st = O.init_state(mps, W, O.Params(chi_max=chi_max, eps=eps), 1)
    return t, st


def _compare(t, st, tol):
    m = O.measure(st)
    assert np.abs(t.measure_sz() - m["sz"]).max() < tol
    assert abs(t.measure_energy() - m["energy"]) < tol
    assert abs(t.measure_norm() - m["norm"]) < tol
    assert t.chi() == O.chi_profile(st)
    _, glam = t.get_mps()
    _, olam = O.global_mps(st)
    for a_, b_ in zip(glam, olam):
        check_spectra(a_, b_, 1e-14, tol)


@pytest.mark.parametrize("L,chi,Delta,steps", [(12, 16, 0.5, 4), (16, 64, 1.0, 3), (14, 128, 1.5, 2)])
def test_step1_matches_oracle(B, L, chi, Delta, steps):
    mps = ti.random_canonical_mps(L, chi, seed=3)
    W = ti.mpo_xxz_nn(L, Delta)
    t, st = _pair(B, mps, W, chi, 1e-14)
    E0 = t.measure_energy()
    for _ in range(steps):
        t.step1(0.05)
        T1.step1(st, 0.05)
        # 1TDVP conserves the energy and the norm at fixed bond dimension
        assert abs(t.measure_energy() - E0) < 1e-10
        assert abs(t.measure_norm() - 1.0) < 1e-11
    _compare(t, st, 1e-9)
    s = t.stats()
    assert s["n_pair"] == 0 and s["kernel_launches"] > 0
    t.close()


def test_step1_long_range_mpo(B):
    """D = 29 exp-sum MPO (configs[3] family): H_eff^(0) over 29 channels."""
    a, lam, _, _ = ti.fit_expsum(100, 9, 2.0)
    L = 12
    W = ti.mpo_xxz_expsum(L, a, lam, 1.0)
    mps = ti.random_canonical_mps(L, 32, seed=4)
    t, st = _pair(B, mps, W, 32, 1e-14)
    for _ in range(2):
        t.step1(0.02)
        T1.step1(st, 0.02)
    _compare(t, st, 1e-9)
    t.close()


def test_hybrid_matches_oracle(B):
    """Neel quench, chi_max = 8: 2TDVP steps until every bond is saturated,
    then 1TDVP; the same integrator sequence and results as the oracle's."""
    L, chi = 12, 8
    W = ti.mpo_xxz_nn(L, 1.0)
    t, st = _pair(B, ti.neel_mps(L), W, chi, 1e-12)
    used_g, used_o = [], []
    trunc = False
    for _ in range(12):
        used_g.append(t.step_hybrid(0.05))
        used_o.append(T1.step_hybrid(st, 0.05))
        trunc = trunc or st.stats.trunc_active
    assert used_g == used_o
    assert used_g[0] == 2 and used_g[-1] == 1
    _compare(t, st, 1e-6 if trunc else 1e-9)
    t.close()


def _pair_p(B, mps, W, chi_max, eps, p, devices=None):
    D_ = max(max(w.shape[0], w.shape[3]) for w in W)
    t = B.Tdvp(len(W), 2, D_, chi_max, devices=devices)
    t.set_params(eps=eps)
    t.set_mpo(W)
    t.set_mps(mps.psi, mps.lam)
    st = O.init_state(mps, W, O.Params(chi_max=chi_max, eps=eps), p)
    return t, st


@pytest.mark.parametrize("p,chi_max", [(2, 16), (4, 16), (2, 64), (4, 64)])
def test_p1tdvp_matches_oracle(B, p, chi_max):
    """Segment-parallel one-site TDVP (tdvp_step1 with n_segments = p,
    reading R-P1TDVP) vs oracle step1p: saturated interiors (chi 16), and
    chi_max above the state's chi so the two-site boundary updates grow their
    bonds (64); the serial p1 case is the tests above."""
    L = 16
    mps = ti.random_canonical_mps(L, 16, seed=12)
    W = ti.mpo_xxz_nn(L, 0.8)
    t, st = _pair_p(B, mps, W, chi_max, 1e-12, p)
    for _ in range(3):
        t.step1(0.05, p)
        T1.step1p(st, 0.05)
    _compare(t, st, 1e-9)
    t.close()


def test_p1tdvp_multi_device_lanes(B):
    """The multi-device executor (segment lanes, repeated device ids on this
    GPU) running the p1TDVP programs, p = 4."""
    L = 16
    mps = ti.random_canonical_mps(L, 16, seed=13)
    W = ti.mpo_xxz_nn(L, 1.0)
    t, st = _pair_p(B, mps, W, 32, 1e-12, 4, devices=[0, 0, 0, 0])
    for _ in range(2):
        t.step1(0.05, 4)
        T1.step1p(st, 0.05)
    _compare(t, st, 1e-9)
    t.close()


def test_hybrid_segments(B):
    """n_segments = 2: 2TDVP (p2) until saturated, then p1TDVP; same sequence
    and results as the oracle's hybrid on the same partition."""
    L, chi = 12, 8
    W = ti.mpo_xxz_nn(L, 1.0)
    t, st = _pair_p(B, ti.neel_mps(L), W, chi, 1e-12, 2)
    used_g, used_o = [], []
    trunc = False
    for _ in range(12):
        used_g.append(t.step_hybrid(0.05, 2))
        used_o.append(T1.step_hybrid(st, 0.05))
        trunc = trunc or st.stats.trunc_active
    assert used_g == used_o and used_g[-1] == 1
    _compare(t, st, 1e-6 if trunc else 1e-9)
    t.close()


def test_step1_rejects_u1(B):
    L = 8
    W = ti.mpo_xxz_nn(L, 1.0)
    t, _ = _pair(B, ti.neel_mps(L), W, 8, 1e-12)
    t.set_params(eps=1e-12, u1=1)
    with pytest.raises(B.TdvpError):
        t.step1(0.05)
    t.close()


@pytest.mark.parametrize("L,chi", [(2, 2), (3, 2), (5, 1), (9, 4)])
def test_step1_edge_shapes(B, L, chi):
    """Shortest chains (one bond; the turnaround site is also the first),
    chi = 1 (a product state stays a product state: the mean-field limit of
    1TDVP), and an odd length."""
    W = ti.mpo_xxz_nn(L, 0.7)
    mps = ti.bloch_mps(L, seed=1) if chi == 1 else ti.random_canonical_mps(L, chi, seed=8)
    t, st = _pair(B, mps, W, chi, 1e-14)
    for _ in range(3):
        t.step1(0.05)
        T1.step1(st, 0.05)
    _compare(t, st, 1e-10)
    if chi == 1:
        assert t.chi() == [1] * (L + 1)
    t.close()


def test_step1_zero_dt_is_identity(B):
    L = 8
    W = ti.mpo_xxz_nn(L, 1.0)
    mps = ti.random_canonical_mps(L, 8, seed=9)
    t, st = _pair(B, mps, W, 8, 1e-14)
    sz0 = O.measure(st)["sz"]
    t.step1(0.0)
    assert np.abs(t.measure_sz() - sz0).max() < 1e-12
    t.close()


def test_step1_bench_workload_invariants(B):
    """bench.py's secondary_1tdvp launch configuration at its full size
    (c5sat: L = 24, chi = 1024 on bonds 10..14, 2048 x 1024 splits through
    the block-Jacobi SVD): properties that hold at any size -- the energy and
    the norm are conserved and no bond grows (a value below eps * sigma_1 may
    be cut by the split's O-7 rule, as in the oracle; the oracle cannot run
    this size in a test)."""
    L, chi = 24, 1024
    mps = ti.random_canonical_mps(L, chi, seed=2)
    W = ti.mpo_xxz_nn(L, 1.0)
    t = B.Tdvp(L, 2, 5, chi)
    t.set_params(eps=1e-12)
    t.set_mpo(W)
    t.set_mps(mps.psi, mps.lam)
    E0, n0, chi0 = t.measure_energy(), t.measure_norm(), t.chi()
    t.step1(0.05)
    assert abs(t.measure_energy() - E0) < 1e-9 * max(1.0, abs(E0))
    assert abs(t.measure_norm() - n0) < 1e-10
    assert all(c <= c0 for c, c0 in zip(t.chi(), chi0))
    assert sum(chi0) - sum(t.chi()) <= 4
    t.close()
