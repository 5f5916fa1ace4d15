"""GPU: U(1) block-sparse splits (tdvp_params.u1, SURVEY §8(f) N1,
PAPER.md:643-651) against the U(1) oracle (oracle/u1.py, pinned equal to the
dense oracle in tests/test_oracle_u1.py) on charge-conserving inputs: Neel
quenches (configs 1/2/3/5 have S^z_tot = 0) and saturated random states of
definite charge, serial and segmented, plus DMRG and the re-gauged dynamic
re-partitioning in U(1) mode."""
import numpy as np
import pytest

import tdvp_inputs as ti
from oracle import dmrg as G
from oracle import tdvp as O

from _parity import check_spectra

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1912_06127_b200 as pkg
    return pkg


def run(B, mps, W, chi_max, eps, dt, steps, p, u1=True, **kw):
    D = max(max(w.shape[0], w.shape[3]) for w in W)
    t = B.Tdvp(len(W), 2, D, chi_max)
    t.set_params(eps=eps, u1=u1, **kw)
    t.set_mpo(W)
    t.set_mps(mps.psi, mps.lam)
    st = O.init_state(mps, W, O.Params(chi_max=chi_max, eps=eps, u1=True), p)
    trunc = False
    for _ in range(steps):
        t.step(dt, p)
        O.step(st, dt)
        trunc = trunc or st.stats.trunc_active
    m = O.measure(st)
    tol = 1e-6 if trunc else 1e-9
    err = max(np.abs(t.measure_sz() - m["sz"]).max(), abs(t.measure_energy() - m["energy"]),
              abs(t.measure_norm() - m["norm"]))
    assert err < tol, err
    psi, lam = t.get_mps()
    _, olam = O.global_mps(st)
    for a, b in zip(lam, olam):
        check_spectra(a, b, eps, tol)
    return t, st, psi, trunc


@pytest.mark.parametrize("p", [1, 2, 4])
def test_u1_neel_quench(B, p):
    L = 32
    t, st, psi, _ = run(B, ti.neel_mps(L), ti.mpo_xxz_nn(L, 0.5), 64, 1e-10, 0.05, 6, p)
    # the evolved tensors keep exact zeros outside their charge blocks
    from oracle import u1 as U
    U.infer_charges(psi)
    t.close()


@pytest.mark.parametrize("p", [1, 2])
def test_u1_saturated_truncated(B, p):
    L = 16
    t, st, _, trunc = run(B, ti.random_u1_mps(L, 32, seed=4), ti.mpo_xxz_nn(L, 1.0), 32, 1e-12, 0.05, 2, p)
    assert trunc
    t.close()


def test_u1_equals_dense_gpu(B):
    """The U(1) and the dense GPU paths agree on a charge-conserving run."""
    L = 24
    mps, W = ti.neel_mps(L), ti.mpo_xxz_nn(L, 1.0)
    out = []
    for u1 in (False, True):
        t = B.Tdvp(L, 2, 5, 64)
        t.set_params(eps=1e-12, u1=u1)
        t.set_mpo(W)
        t.set_mps(mps.psi, mps.lam)
        for _ in range(5):
            t.step(0.05, 2)
        out.append((t.measure_sz(), t.measure_energy()))
        t.close()
    assert np.abs(out[0][0] - out[1][0]).max() < 1e-9 and abs(out[0][1] - out[1][1]) < 1e-9


def test_u1_dmrg(B):
    L = 12
    W = ti.mpo_xxz_nn(L, 0.5)
    mps = ti.neel_mps(L)
    t = B.Tdvp(L, 2, 5, 64)
    t.set_params(eps=1e-12, u1=True)
    t.set_mpo(W)
    t.set_mps(mps.psi, mps.lam)
    E = t.dmrg(3, 4)
    _, Eo = G.dmrg(mps, W, O.Params(chi_max=64, eps=1e-12, u1=True), 3, 4)
    assert np.abs(np.array(E) - np.array(Eo)).max() < 1e-9
    psi, _ = t.get_mps()
    from oracle import u1 as U
    U.infer_charges(psi)  # the re-gauged result keeps its block structure
    t.close()


def test_u1_rebalance(B):
    L, p = 32, 4
    t, st, psi, _ = run(B, ti.neel_mps(L), ti.mpo_xxz_nn(L, 0.5), 64, 1e-12, 0.05, 1, p, rebalance=0.05)
    t.close()


def test_u1_rejects_charge_indefinite_state(B):
    L = 8
    t = B.Tdvp(L, 2, 5, 16)
    t.set_params(u1=True)
    t.set_mpo(ti.mpo_xxz_nn(L, 1.0))
    m = ti.random_canonical_mps(L, 8, seed=1)  # dense random tensors: no definite charge
    t.set_mps(m.psi, m.lam)
    with pytest.raises(Exception):
        t.step(0.05, 1)
    t.close()
