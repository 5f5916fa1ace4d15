"""Pins of the two-site DMRG oracle (oracle/dmrg.py) against
things other than itself: dense eigendecompositions, an exact Krylov
breakdown, exact diagonalisation of the chain, the free-fermion closed form,
and the variational principle.  CPU only."""
import numpy as np
import pytest

import tdvp_inputs as ti
from oracle import dense as D
from oracle import dmrg as G
from oracle import tdvp as O

NN = lambda r: 1.0 if r == 1 else 0.0  # noqa: E731


def test_lanczos_ground_vs_dense():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((40, 40)) + 1j * rng.standard_normal((40, 40))
    H = (A + A.conj().T) / 2
    v = rng.standard_normal(40) + 1j * rng.standard_normal(40)
    x, e = G.lanczos_ground(lambda y: H @ y, v, K=8, restarts=40)
    w, U = np.linalg.eigh(H)
    assert abs(e - w[0]) < 1e-10
    assert abs(abs(np.vdot(U[:, 0], x)) - 1.0) < 1e-8
    assert abs(np.linalg.norm(x) - 1.0) < 1e-14


def test_lanczos_ground_exact_on_invariant_subspace():
    """6 distinct eigenvalues < K = 8: the Krylov space is the whole space
    after 6 steps (breakdown), so one restart is exact."""
    d = np.array([0.7, -1.3, 2.0, 0.1, -0.4, 1.1])
    v = np.ones(6, complex)
    x, e = G.lanczos_ground(lambda y: d * y, v, K=8, restarts=1)
    assert abs(e - d.min()) < 1e-14
    ref = np.zeros(6)
    ref[np.argmin(d)] = 1.0
    assert np.abs(np.abs(x) - ref).max() < 1e-12
    assert x[np.argmin(d)].real > 0  # sign convention: y_0 = <v_1|x> >= 0


@pytest.mark.parametrize("Delta", [0.5, 1.0])
def test_dmrg_l10_equals_exact_diagonalisation(Delta):
    L = 10
    W = ti.mpo_xxz_nn(L, Delta)
    st, E = G.dmrg(ti.neel_mps(L), W, O.Params(chi_max=32, eps=1e-12), n_sweeps=4, restarts=4)
    Hd = D.dense_hamiltonian(L, NN, Delta)
    Hd = Hd.toarray() if hasattr(Hd, "toarray") else np.asarray(Hd)
    e_ed = np.linalg.eigvalsh(Hd)[0]
    assert abs(E[-1] - e_ed) < 1e-9, (E, e_ed)
    m = O.measure(st)
    assert abs(m["energy"] - e_ed) < 1e-9
    assert np.abs(m["sz"]).max() < 1e-8  # non-degenerate S^z_tot = 0 ground state, spin-flip symmetric
    assert all(E[k + 1] <= E[k] + 1e-12 for k in range(len(E) - 1))  # variational


def test_dmrg_free_fermions():
    """Delta = 0: H = (J/2) sum (c+_i c_{i+1} + h.c.) by Jordan-Wigner; the
    S^z_tot = 0 ground energy is the sum of the L/2 lowest single-particle
    energies.  DMRG (chi_max = 64 truncates a critical chain) is variational."""
    L = 24
    W = ti.mpo_xxz_nn(L, 0.0)
    st, E = G.dmrg(ti.neel_mps(L), W, O.Params(chi_max=64, eps=1e-12), n_sweeps=4, restarts=3)
    h = np.diag(np.full(L - 1, 0.5), 1) + np.diag(np.full(L - 1, 0.5), -1)
    e_ff = np.sort(np.linalg.eigvalsh(h))[: L // 2].sum()
    m = O.measure(st)
    assert m["energy"] >= e_ff - 1e-10
    assert m["energy"] - e_ff < 1e-6, (m["energy"], e_ff)
