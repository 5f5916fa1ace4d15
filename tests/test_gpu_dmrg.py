"""GPU: two-site DMRG (tdvp_dmrg) against the DMRG oracle
(oracle/dmrg.py) on the same seeded inputs, sweep by sweep, and the paper's
quench protocol: DMRG ground state of one Hamiltonian, then 2TDVP under
another."""
import numpy as np
import pytest

import tdvp_inputs as ti
from oracle import dense as D
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


def gpu_dmrg(B, mps, W, chi_max, eps, sweeps, restarts):
    D_ = max(max(w.shape[0], w.shape[3]) for w in W)
    t = B.Tdvp(len(W), 2, D_, chi_max)
    t.set_params(eps=eps)
    t.set_mpo(W)
    t.set_mps(mps.psi, mps.lam)
    E = t.dmrg(sweeps, restarts)
    return t, E


@pytest.mark.parametrize("case", ["xxz10", "xxx10", "ff24", "lr12"])
def test_dmrg_matches_oracle(B, case):
    if case == "ff24":
        L, W, chi, sweeps = 24, ti.mpo_xxz_nn(24, 0.0), 64, 4  # chi_max binds from sweep 3
    elif case == "lr12":
        a, lam, _, _ = ti.fit_expsum(100, 9, 2.0)
        L, W, chi, sweeps = 12, ti.mpo_xxz_expsum(12, a, lam, 1.0), 32, 3
    else:
        L, W, chi, sweeps = 10, ti.mpo_xxz_nn(10, 0.5 if case == "xxz10" else 1.0), 32, 4
    mps = ti.neel_mps(L)
    t, E = gpu_dmrg(B, mps, W, chi, 1e-12, sweeps, 4)
    st, Eo = G.dmrg(mps, W, O.Params(chi_max=chi, eps=1e-12), sweeps, 4)
    tol = 1e-6 if st.stats.trunc_active else 1e-9
    assert np.abs(np.array(E) - np.array(Eo)).max() < tol, (E, Eo)
    m = O.measure(st)
    assert np.abs(t.measure_sz() - m["sz"]).max() < tol
    assert abs(t.measure_energy() - m["energy"]) < tol
    _, glam = t.get_mps()
    psi, lam_o = O.global_mps(st)
    olam = ti.canonicalize(O._chain_tensors(psi, lam_o)).lam  # tdvp_dmrg re-gauges its result
    for a_, b_ in zip(glam, olam):
        check_spectra(a_, b_, 1e-12, tol)
    if L <= 12:
        NN = (lambda r: 1.0 if r == 1 else 0.0) if case != "lr12" else (lambda r: float(ti.expsum_J(a, lam, [r])[0]))
        Hd = D.dense_hamiltonian(L, NN, 0.5 if case == "xxz10" else 1.0)
        Hd = Hd.toarray() if hasattr(Hd, "toarray") else np.asarray(Hd)
        assert abs(t.measure_energy() - np.linalg.eigvalsh(Hd)[0]) < 1e-8
    t.close()


def test_dmrg_ground_state_quench(B):
    """Ground state of XXZ Delta = 0.5 by DMRG (unique, finite-size gap ~ 1/L;
    not Delta > 1, whose two near-degenerate Neel-like states make any DMRG's
    superposition rounding-dependent), then 2TDVP under Delta = 1.5 (a quench,
    PAPER.md:130), p = 2 segments; GPU vs oracle."""
    L, chi, dt = 16, 64, 0.05
    W0, W1 = ti.mpo_xxz_nn(L, 0.5), ti.mpo_xxz_nn(L, 1.5)
    mps = ti.neel_mps(L)
    t, _ = gpu_dmrg(B, mps, W0, chi, 1e-12, 3, 3)
    st, _ = G.dmrg(mps, W0, O.Params(chi_max=chi, eps=1e-12), 3, 3)
    t.set_mpo(W1)
    # tdvp_dmrg re-gauges its final state into inverse-canonical form (the
    # quench input must be): the same exact re-gauging here
    psi, lam = O.global_mps(st)
    st2 = O.init_state(ti.canonicalize(O._chain_tensors(psi, lam)), W1, O.Params(chi_max=chi, eps=1e-12), 2)
    trunc = st.stats.trunc_active
    for _ in range(4):
        t.step(dt, 2)
        O.step(st2, dt)
        trunc = trunc or st2.stats.trunc_active
    m = O.measure(st2)
    tol = 1e-6 if trunc else 1e-9
    assert np.abs(t.measure_sz() - m["sz"]).max() < tol
    assert abs(t.measure_energy() - m["energy"]) < tol
    t.close()
