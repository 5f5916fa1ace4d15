"""Pins of the U(1) block-sparse oracle path (oracle/u1.py, Params.u1;
SURVEY.md §8(f) N1) against the DENSE oracle, which is
itself pinned (tests/test_oracle_pins.py): for charge-conserving inputs the
sector-wise SVD is the dense SVD reordered, so the U(1) integrator must
reproduce the dense one; and the tracked bond charges must equal the ones
the nonzero structure of the evolved state implies.  CPU only."""
import numpy as np
import pytest

import tdvp_inputs as ti
from oracle import dmrg as G
from oracle import tdvp as O
from oracle import u1 as U


def _block_theta(rng, qa, qb, d=2):
    cl, cr = len(qa), len(qb)
    t = np.zeros((cl, d, d, cr), dtype=np.complex128)
    for s1 in range(d):
        for s2 in range(d):
            mask = (qa[:, None] + U.C_S[s1]) == (qb[None, :] - U.C_S[s2])
            t[:, s1, s2, :] = np.where(mask, rng.standard_normal(mask.shape) + 1j * rng.standard_normal(mask.shape), 0)
    return t


@pytest.mark.parametrize("chi_max,eps", [(100, 1e-12), (9, 1e-12), (5, 1e-10), (1, 1e-12)])
def test_svd_u1_equals_dense(chi_max, eps):
    rng = np.random.default_rng(chi_max)
    qa = np.array([0, 2, 2, -2, 0, 4, -2, 0])
    qb = np.array([0, 0, 2, -2, 2, 0, -4])
    for trial in range(20):
        th = _block_theta(rng, qa, qb) * np.exp(-rng.uniform(0, 10))
        p = O.Params(chi_max=chi_max, eps=eps)
        pl, S, pr, w, r, ce = O.svd_truncate(th, p)
        pl1, S1, pr1, w1, r1, ce1, qm = U.svd_truncate_u1(th, qa, qb, p)
        k = len(S)
        assert len(S1) == k and np.allclose(S1, S, rtol=1e-12, atol=1e-14 * S[0])
        assert abs(w1 - w) <= 1e-12 * np.sum(np.abs(th) ** 2)
        M = th.reshape(len(qa) * 2, 2 * len(qb))
        rec = pl.reshape(-1, k) @ np.diag(1 / S) @ pr.reshape(k, -1)
        rec1 = pl1.reshape(-1, k) @ np.diag(1 / S1) @ pr1.reshape(k, -1)
        assert np.linalg.norm(rec1 - rec) <= 1e-10 * np.linalg.norm(M)
        # every kept vector lives in its charge sector
        rq = (qa[:, None] + U.C_S[None, :]).reshape(-1)
        cq = (qb[None, :] - U.C_S[:, None]).reshape(-1)
        for c in range(k):
            assert np.all(pl1.reshape(-1, k)[rq != qm[c], c] == 0)
            assert np.all(pr1.reshape(k, -1)[c, cq != qm[c]] == 0)


@pytest.mark.parametrize("p", [1, 2])
def test_u1_integrator_equals_dense_untruncated(p):
    L = 12
    W = ti.mpo_xxz_nn(L, 0.5)
    mps = ti.neel_mps(L)
    a = O.init_state(mps, W, O.Params(chi_max=64, eps=1e-12), p)
    b = O.init_state(mps, W, O.Params(chi_max=64, eps=1e-12, u1=True), p)
    for _ in range(6):
        O.step(a, 0.05)
        O.step(b, 0.05)
    ma, mb = O.measure(a), O.measure(b)
    assert np.abs(ma["sz"] - mb["sz"]).max() < 1e-12
    assert abs(ma["energy"] - mb["energy"]) < 1e-12
    psi, lam = O.global_mps(b)
    q = U.infer_charges(psi)
    for seg in b.segs:
        for k in range(seg.s + 1, seg.e + 1):
            assert np.array_equal(q[k], seg.qb[k])


def test_u1_integrator_equals_dense_truncated():
    """chi_max binding on a saturated U(1) state: same kept spectra, same observables."""
    L = 12
    W = ti.mpo_xxz_nn(L, 1.0)
    mps = ti.random_u1_mps(L, 16, seed=5)
    a = O.init_state(mps, W, O.Params(chi_max=16, eps=1e-12), 2)
    b = O.init_state(mps, W, O.Params(chi_max=16, eps=1e-12, u1=True), 2)
    for _ in range(2):
        O.step(a, 0.05)
        O.step(b, 0.05)
    assert b.stats.trunc_active
    ma, mb = O.measure(a), O.measure(b)
    assert np.abs(ma["sz"] - mb["sz"]).max() < 1e-10
    _, la = O.global_mps(a)
    _, lb = O.global_mps(b)
    for x, y in zip(la, lb):
        assert len(x) == len(y) and np.allclose(x, y, atol=1e-11 * x[0])


def test_u1_dmrg_equals_dense():
    L = 10
    W = ti.mpo_xxz_nn(L, 0.5)
    _, E = G.dmrg(ti.neel_mps(L), W, O.Params(chi_max=32, eps=1e-12), 3, 4)
    _, E1 = G.dmrg(ti.neel_mps(L), W, O.Params(chi_max=32, eps=1e-12, u1=True), 3, 4)
    assert np.abs(np.array(E) - np.array(E1)).max() < 1e-10
