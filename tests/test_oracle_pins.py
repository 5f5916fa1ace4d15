"""Pins of the CPU oracle against things other than itself.

Every pin compares the oracle with an exact reference derived from the
paper's definitions and the mathematics: dense exponentials, closed forms,
invariants, and special cases.  CPU only.
"""
import numpy as np
import pytest
import scipy.linalg

import tdvp_inputs as ti
from oracle import dense as D
from oracle import tdvp as O

NN = lambda r: 1.0 if r == 1 else 0.0  # noqa: E731


def dense_of(st_or_mps):
    if isinstance(st_or_mps, O.State):
        psi, lam = O.global_mps(st_or_mps)
    else:
        psi, lam = st_or_mps.psi, st_or_mps.lam
    return O.to_dense(psi, lam)


def mpo_dense(W):
    """Contract an MPO to a dense matrix (test helper, independent of oracle)."""
    T = W[0][0]  # (d, d, D)
    T = np.transpose(T, (2, 0, 1))  # (D, s, t)
    for j in range(1, len(W)):
        Wj = W[j]  # (Dl, s, t, Dr)
        n = T.shape[1]
        T = np.einsum("wab,wstv->vasbt", T, Wj).reshape(Wj.shape[3], n * 2, n * 2)
    return T[0]


# --------------------------------------------------------------------------
# inputs pinned to the model definition
# --------------------------------------------------------------------------

@pytest.mark.parametrize("Delta", [0.0, 0.5, 1.5])
def test_mpo_nn_equals_dense_model(Delta):
    L = 6
    Hm = mpo_dense(ti.mpo_xxz_nn(L, Delta))
    Hd = D.dense_hamiltonian(L, NN, Delta)
    assert np.abs(Hm - Hd).max() < 1e-14


def test_mpo_expsum_equals_dense_model():
    L = 7
    a, lam = [0.3, 1.1], [0.5, -0.2]
    Hm = mpo_dense(ti.mpo_xxz_expsum(L, a, lam, 0.8))
    Hd = D.dense_hamiltonian(L, lambda r: float(ti.expsum_J(a, lam, [r])[0]), 0.8)
    assert np.abs(Hm - Hd).max() < 1e-13


def test_expsum_fit_quality():
    # 1/r^2 by 9 exponentials on r = 1..100 (AMB-12)
    a, lam, abs_err, rel_err = ti.fit_expsum(100, 9, 2.0)
    assert np.all((lam > 0) & (lam < 1))
    assert abs_err < 1e-7 and rel_err < 1e-3
    assert ti.mpo_xxz_expsum(10, a, lam, 1.0)[3].shape == (29, 2, 2, 29)


def test_random_canonical_mps_is_inverse_canonical():
    mps = ti.random_canonical_mps(10, 8, seed=3)
    v = dense_of(mps)
    assert abs(np.linalg.norm(v) - 1) < 1e-12
    # every Psi_j is an orthogonality centre: ||Psi_j||_F = 1
    for p in mps.psi:
        assert abs(np.linalg.norm(p) - 1) < 1e-12
    # Lambda_j are the Schmidt values of the dense state
    for j, lam in enumerate(mps.lam):
        s = np.linalg.svd(v.reshape(2 ** (j + 1), -1), compute_uv=False)
        assert np.allclose(s[: len(lam)], lam, atol=1e-12)


# --------------------------------------------------------------------------
# P9 Lanczos, P15 SVD truncation
# --------------------------------------------------------------------------

def test_p9_lanczos_vs_dense_exp():
    rng = np.random.default_rng(7)
    A = rng.standard_normal((32, 32)) + 1j * rng.standard_normal((32, 32))
    H = (A + A.conj().T) / 2
    H /= np.linalg.norm(H, 2)
    v = rng.standard_normal(32) + 1j * rng.standard_normal(32)
    tau = -0.05j
    ref = scipy.linalg.expm(tau * H) @ v
    out = O.expm_lanczos(lambda x: H @ x, v, tau, K=8)
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) < 1e-10
    # norm preserved for imaginary tau
    assert abs(np.linalg.norm(out) - np.linalg.norm(v)) < 1e-13 * np.linalg.norm(v)


def test_p9_lanczos_special_cases():
    Hd = np.diag([1.0, 2.0]).astype(complex)
    out = O.expm_lanczos(lambda x: Hd @ x, np.array([1.0, 0.0], complex), -0.1j)
    assert np.allclose(out, [np.exp(-0.1j), 0.0], atol=1e-15)
    rng = np.random.default_rng(1)
    v = rng.standard_normal(10) + 1j * rng.standard_normal(10)
    A = rng.standard_normal((10, 10))
    H = A + A.T
    info = {}
    assert np.allclose(O.expm_lanczos(lambda x: H @ x, v, 0.0, info=info), v, atol=1e-13)
    # invariant subspace smaller than K -> breakdown -> exact
    H4 = np.diag([0.3, -1.2, 2.0, 0.7]).astype(complex)
    v4 = np.ones(4, complex)
    info = {}
    out = O.expm_lanczos(lambda x: H4 @ x, v4, -0.7j, K=8, info=info)
    assert info["breakdown"] and info["k"] == 4
    assert np.allclose(out, np.exp(-0.7j * np.diag(H4)) * v4, atol=1e-13)


def test_p9b_paper_mode_krylov_stop_rule():
    """Paper-mode Krylov ("maximum of 8 basis vectors ...
    convergence tolerance 1e-6"; SURVEY O-10 step 5, AMB-5): with tol > 0 the
    oracle stops after the first m with n0 beta_m |(exp(tau T_m) e_1)_m| < tol.

    Pinned on a case whose Lanczos process is known in closed form: for a real
    symmetric tridiagonal (Jacobi) matrix J and v = n0 e_1, the Lanczos basis
    is e_1, e_2, ... and T_m is J's leading m x m block.  So the stopping index
    is predicted here from scipy.linalg.expm of the leading blocks (an
    independent route: Pade, not the oracle's eigh), and the result must be
    n0 * expm(tau T_m) e_1 embedded in R^n, within tol of the exact
    n0 * expm(tau J) e_1.  An off-by-one in the index, a missing n0 or a
    wrong component of c moves K_eff or the result."""
    rng = np.random.default_rng(5)
    n, n0 = 40, 3.0
    alpha = rng.uniform(-1.0, 1.0, n)
    beta = rng.uniform(0.5, 1.5, n - 1)
    J = np.diag(alpha) + np.diag(beta, 1) + np.diag(beta, -1)
    v = np.zeros(n, complex)
    v[0] = n0
    for tau, tol in ((-0.05j, 1e-6), (-0.2j, 1e-6), (0.1j, 1e-7), (-0.02j, 1e-12), (-0.5j, 1e-6)):
        pred = None
        for m in range(1, 9):
            c_m = scipy.linalg.expm(tau * J[:m, :m])[m - 1, 0]
            if n0 * beta[m - 1] * abs(c_m) < tol:
                pred = m
                break
        info = {}
        out = O.expm_lanczos(lambda x: J @ x, v, tau, K=8, tol=tol, info=info)
        k_eff = info["k"]
        assert k_eff == (pred if pred is not None else 8), (tau, tol, k_eff, pred)
        ref_k = np.zeros(n, complex)
        ref_k[:k_eff] = n0 * scipy.linalg.expm(tau * J[:k_eff, :k_eff])[:, 0]
        assert np.abs(out - ref_k).max() < 1e-13
        exact = n0 * scipy.linalg.expm(tau * J)[:, 0]
        assert np.linalg.norm(out - exact) < (10 * tol if pred is not None else 1e-6)
    # an easy spectrum stops early (K_eff < K); a generic Hermitian case is within tol
    assert O.expm_lanczos(lambda x: J @ x, v, -0.05j, K=8, tol=1e-6, info=(inf := {})) is not None and inf["k"] < 8
    A = rng.standard_normal((32, 32)) + 1j * rng.standard_normal((32, 32))
    H = (A + A.conj().T) / 2
    H /= np.linalg.norm(H, 2)
    x = rng.standard_normal(32) + 1j * rng.standard_normal(32)
    info = {}
    out = O.expm_lanczos(lambda y: H @ y, x, -0.05j, K=8, tol=1e-6, info=info)
    assert info["k"] < 8
    assert np.linalg.norm(out - scipy.linalg.expm(-0.05j * H) @ x) < 1e-6


def test_p15_svd_tail_and_reconstruction():
    rng = np.random.default_rng(11)
    for trial in range(200):
        m, n = rng.integers(2, 20, size=2)
        M = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
        M *= rng.uniform(0.1, 10)
        chi_max = int(rng.integers(1, min(m, n) + 1))
        p = O.Params(chi_max=chi_max, eps=1e-12)
        th = M.reshape(m, 1, 1, n)
        pl, S, pr, w, r, _ = O.svd_truncate(th, p)
        s_ref = np.linalg.svd(M, compute_uv=False)  # independent routine
        chi = len(S)
        assert abs(w - np.sum(s_ref[chi:] ** 2)) <= 1e-10 * np.sum(s_ref ** 2)
        assert np.allclose(S, s_ref[:chi], rtol=1e-12, atol=1e-14 * s_ref[0])
        # Psi_L V Psi_R reproduces the truncated matrix; Psi_L / S has orthonormal columns
        U = pl.reshape(m, chi) / S[None, :]
        assert np.allclose(U.conj().T @ U, np.eye(chi), atol=1e-12)
        rec = pl.reshape(m, chi) @ np.diag(1 / S) @ pr.reshape(chi, n)
        assert abs(np.linalg.norm(M - rec) ** 2 - w) <= 1e-10 * np.linalg.norm(M) ** 2


def test_truncation_rules():
    # diag(1, 1e-13), eps = 1e-12 -> chi = 1, w = 1e-26 (SPEC.md linalg-core example)
    th = np.diag([1.0, 1e-13]).astype(complex).reshape(2, 1, 1, 2)
    _, S, _, w, _, _ = O.svd_truncate(th, O.Params(chi_max=2, eps=1e-12))
    assert len(S) == 1 and abs(w - 1e-26) < 1e-40
    sig = np.array([1.0, 0.5, 0.5, 0.5 * (1 - 1e-8), 0.1, 1e-3])
    # multiplet guard: cut at 3 would split the degenerate triple -> chi = 1 (AMB-9)
    assert O.truncation_rank(sig, O.Params(chi_max=3)) == 1
    assert O.truncation_rank(sig, O.Params(chi_max=4)) == 4
    # w_max rule: minimum chi with tail <= w_max
    assert O.truncation_rank(sig, O.Params(chi_max=6, w_max=1e-6 * 1.01)) == 5
    assert O.truncation_rank(sig, O.Params(chi_max=6, w_max=0.0101 + 1e-6)) == 4
    # eps rule
    assert O.truncation_rank(sig, O.Params(chi_max=6, eps=2e-3)) == 5
    # R-9b: a numerically degenerate pair (gap < 1e-13 sigma_1) straddling the eps cut is dropped whole
    sig2 = np.array([1.0, 0.2, 1.0e-12 + 3e-14, 1.0e-12 - 2e-14, 5e-13])
    assert O.truncation_rank(sig2, O.Params(chi_max=5, eps=1e-12)) == 2
    sig3 = np.array([1.0, 0.2, 1.0e-12 + 3e-13, 1.0e-12 - 2e-14, 5e-13])
    assert O.truncation_rank(sig3, O.Params(chi_max=5, eps=1e-12)) == 3


# --------------------------------------------------------------------------
# P7 env closure, P8 H_eff = P^dagger H P
# --------------------------------------------------------------------------

def _left_basis(psi, lam, j):
    """Left basis |Phi_L> of sites < j: Psi_0 V_0 ... Psi_{j-1} V_{j-1}."""
    v = np.ones((1, 1), complex)
    for k in range(j):
        A = psi[k] * (1 / lam[k])[None, None, :]
        v = np.tensordot(v, A, axes=(1, 0)).reshape(-1, A.shape[2])
    return v  # (2^j, chi)


def _right_basis(psi, lam, j):
    """Right basis of sites > j: V_j Psi_{j+1} V_{j+1} ... Psi_{L-1} -> (chi_j, 2^(L-1-j))."""
    L = len(psi)
    v = np.ones((1, 1), complex)
    for k in range(L - 1, j, -1):
        B = (1 / lam[k - 1])[:, None, None] * psi[k]
        v = np.tensordot(B, v, axes=(2, 0)).reshape(B.shape[0], -1)
    return v


def test_p8_heff_two_site_is_projected_hamiltonian():
    L, j = 6, 2
    mps = ti.random_canonical_mps(L, 4, seed=4)
    W = ti.mpo_xxz_expsum(L, [0.7, 0.4], [0.5, 0.1], 1.3)
    H = mpo_dense(W)
    beta, gamma = O._mps_envs(mps.psi, mps.lam, W)
    PL = _left_basis(mps.psi, mps.lam, j)         # (2^j, cl)
    PR = _right_basis(mps.psi, mps.lam, j + 1)    # (cr, 2^(L-j-2))
    cl, cr = PL.shape[1], PR.shape[0]
    P = np.einsum("xa,su,bz->xszaub", PL, np.eye(4), PR).reshape(2 ** L, cl * 4 * cr)
    Heff_ref = P.conj().T @ H @ P
    n = cl * 4 * cr
    Heff = np.zeros((n, n), complex)
    for k in range(n):
        e = np.zeros(n, complex)
        e[k] = 1
        Heff[:, k] = O.apply_h2(beta[j], W[j], W[j + 1], gamma[j + 1], e.reshape(cl, 2, 2, cr)).reshape(-1)
    assert np.abs(Heff - Heff_ref).max() < 1e-12
    assert np.abs(Heff - Heff.conj().T).max() < 1e-12


def test_p8_heff_one_site_is_projected_hamiltonian():
    L, j = 6, 3
    mps = ti.random_canonical_mps(L, 4, seed=6)
    W = ti.mpo_xxz_nn(L, 0.6)
    H = mpo_dense(W)
    beta, gamma = O._mps_envs(mps.psi, mps.lam, W)
    PL = _left_basis(mps.psi, mps.lam, j)
    PR = _right_basis(mps.psi, mps.lam, j)
    cl, cr = PL.shape[1], PR.shape[0]
    P = np.einsum("xa,su,bz->xszaub", PL, np.eye(2), PR).reshape(2 ** L, cl * 2 * cr)
    Heff_ref = P.conj().T @ H @ P
    n = cl * 2 * cr
    Heff = np.stack([O.apply_h1(beta[j], W[j], gamma[j], np.eye(n)[k].reshape(cl, 2, cr).astype(complex)).reshape(-1)
                     for k in range(n)], axis=1)
    assert np.abs(Heff - Heff_ref).max() < 1e-12


def test_p7_env_closure_equals_energy():
    L = 8
    mps = ti.random_canonical_mps(L, 8, seed=8)
    a, lam = [0.6, 0.3], [0.7, 0.2]
    W = ti.mpo_xxz_expsum(L, a, lam, 0.9)
    v = dense_of(mps)
    Hd = D.dense_hamiltonian(L, lambda r: float(ti.expsum_J(a, lam, [r])[0]), 0.9)
    E = np.vdot(v, Hd @ v).real
    beta, gamma = O._mps_envs(mps.psi, mps.lam, W)
    for j in range(L - 1):
        th = O.merge_theta(mps.psi[j], 1 / mps.lam[j], mps.psi[j + 1])
        e2 = np.vdot(th, O.apply_h2(beta[j], W[j], W[j + 1], gamma[j + 1], th)).real
        e1 = np.vdot(mps.psi[j], O.apply_h1(beta[j], W[j], gamma[j], mps.psi[j])).real
        assert abs(e2 - E) < 1e-10 and abs(e1 - E) < 1e-10
    m = O.measure((mps.psi, mps.lam), W)
    assert abs(m["energy"] - E) < 1e-10
    assert np.allclose(m["sz"], D.sz_dense(v, L), atol=1e-12)


# --------------------------------------------------------------------------
# P1, P2: exact small chains; literal serial sweep == App. A program at p=1
# --------------------------------------------------------------------------

@pytest.mark.parametrize("L", [2, 3, 4, 5])
def test_p1_p2_full_rank_step_is_exact(L):
    # every local space is the full Hilbert space, so every substep is an exact
    # exponential and the exponents sum to -dt (eq:proj2site term counts)
    mps = ti.random_canonical_mps(L, 64, seed=5)
    W = ti.mpo_xxz_nn(L, 0.7)
    H = D.dense_hamiltonian(L, NN, 0.7)
    st = O.init_state(mps, W, O.Params(chi_max=64), 1)
    v0 = dense_of(mps)
    for n in range(3):
        O.step(st, 0.05)
        v0 = D.evolve(H, v0, 0.05)
        assert np.abs(dense_of(st) - v0).max() < 1e-11


def test_literal_serial_equals_appendix_program():
    L = 9
    mps = ti.neel_mps(L)
    W = ti.mpo_xxz_nn(L, 0.4)
    p = O.Params(chi_max=5, eps=1e-10)
    st = O.init_state(mps, W, p, 1)
    psi, lam = [x.copy() for x in mps.psi], [x.copy() for x in mps.lam]
    beta, gamma = O._mps_envs(psi, lam, W)
    for n in range(6):
        O.step(st, 0.1)
        O.serial_step_literal(psi, lam, W, beta, gamma, 0.1, p)
    gpsi, glam = O.global_mps(st)
    for a, b in zip(glam, lam):
        assert np.array_equal(a, b)
    for a, b in zip(gpsi, psi):
        assert np.array_equal(a, b)


# --------------------------------------------------------------------------
# P3, P4, P5: config 1 against exact diagonalisation; conservation laws
# --------------------------------------------------------------------------

def test_p3_p4_p5_config1_vs_ed():
    cfg = ti.config("c1")
    L = cfg["L"]
    H = D.dense_hamiltonian(L, NN, 1.0)
    v0 = dense_of(cfg["mps"])
    errs = []
    for dt in (0.05, 0.025):
        st = O.init_state(cfg["mps"], cfg["mpo"], O.Params(chi_max=32, eps=1e-12), 1)
        E0 = O.measure(st)["energy"]
        for _ in range(int(round(1.0 / dt))):
            O.step(st, dt)
        m = O.measure(st)
        ref = D.sz_dense(D.evolve(H, v0, 1.0), L)
        errs.append(np.abs(m["sz"] - ref).max())
        assert abs(m["norm"] - 1) < 1e-12                 # P4
        assert abs(m["energy"] - E0) < 1e-10              # P5
        assert abs(E0 - np.vdot(v0, H @ v0).real) < 1e-14
    assert errs[0] < 1e-6                                 # P3
    assert errs[0] / errs[1] > 3.5                        # at least second order in dt


# --------------------------------------------------------------------------
# P6 time reversal, P10 free fermions, P11 one-body exactness,
# P12 invariance, P13 serial vs segmented, P14 magnon sectors
# --------------------------------------------------------------------------

def test_p6_time_reversal_untruncated():
    L = 8
    mps = ti.neel_mps(L)
    st = O.init_state(mps, ti.mpo_xxz_nn(L, 0.5), O.Params(chi_max=64), 1)
    for _ in range(3):
        O.step(st, 0.1)
    for _ in range(3):
        O.step(st, -0.1)
    v, v0 = dense_of(st), dense_of(mps)
    assert 1 - abs(np.vdot(v, v0)) / np.linalg.norm(v) < 1e-12


@pytest.mark.parametrize("p", [1, 2])
def test_p10_free_fermion_closed_form(p):
    L, T = 16, 0.6
    up = [i for i in range(L) if i % 2 == 0]
    ref = D.free_fermion_sz(L, T, up)
    errs = []
    for dt in (0.1, 0.05):
        st = O.init_state(ti.neel_mps(L), ti.mpo_xxz_nn(L, 0.0), O.Params(chi_max=64, eps=1e-12), p)
        for _ in range(int(round(T / dt))):
            O.step(st, dt)
        m = O.measure(st)
        errs.append(np.abs(m["sz"] - ref).max())
        # E = 0 conserved: exactly for serial, up to the parallel error for p > 1
        assert abs(m["energy"]) < (1e-10 if p == 1 else 1e-8)
    assert errs[1] < errs[0] and errs[1] < 1e-5


@pytest.mark.parametrize("p", [1, 2, 4])
def test_p11_one_body_is_exact(p):
    L, h = 8, 0.7
    st = O.init_state(ti.neel_mps(L), ti.mpo_onsite(L, h * ti.SX), O.Params(chi_max=8), p)
    for _ in range(10):
        O.step(st, 0.1)
    exact = np.array([0.5 if i % 2 == 0 else -0.5 for i in range(L)]) * np.cos(h * 1.0)
    assert np.abs(O.measure(st)["sz"] - exact).max() < 1e-12


@pytest.mark.parametrize("p", [1, 2, 4])
def test_p12_invariance(p):
    L = 8
    st = O.init_state(ti.all_up_mps(L), ti.mpo_xxz_nn(L, 1.3), O.Params(chi_max=8), p)
    for _ in range(4):
        O.step(st, 0.1)
    assert np.abs(O.measure(st)["sz"] - 0.5).max() < 1e-13
    mps = ti.random_canonical_mps(L, 4, seed=9)
    st = O.init_state(mps, ti.mpo_zero(L), O.Params(chi_max=16), p)
    for _ in range(3):
        O.step(st, 0.1)
    v, v0 = dense_of(st), dense_of(mps)
    assert np.abs(v - v0).max() < 1e-13


@pytest.mark.parametrize("p", [2, 4])
def test_p13_segmented_converges_to_serial(p):
    L, T = 12, 0.4
    W = ti.mpo_xxz_nn(L, 0.5)
    devs = []
    for dt in (0.04, 0.02, 0.01):
        out = []
        for pp in (1, p):
            st = O.init_state(ti.neel_mps(L), W, O.Params(chi_max=64), pp)
            for _ in range(int(round(T / dt))):
                O.step(st, dt)
            out.append(O.measure(st)["sz"])
        devs.append(np.abs(out[0] - out[1]).max())
    assert devs[0] > devs[1] > devs[2]
    assert devs[2] < 1e-9


@pytest.mark.parametrize("p", [1, 2])
def test_p14_magnon_sector(p):
    L = 16
    errs = []
    for dt in (0.1, 0.05):
        st = O.init_state(ti.single_flip_mps(L, [7, 8]), ti.mpo_xxz_nn(L, 0.5), O.Params(chi_max=16), p)
        for _ in range(int(round(1.0 / dt))):
            O.step(st, dt)
        ref = D.magnon_sz(L, 2, NN, 0.5, [7, 8], 1.0)
        errs.append(np.abs(O.measure(st)["sz"] - ref).max())
    assert errs[1] < 1e-4
    assert 3.0 < errs[0] / errs[1] < 5.5  # second order


@pytest.mark.parametrize("p", [1, 2])
def test_single_magnon_long_range(p):
    # chi = 2 one-magnon superposition under an exp-sum long-range XXZ MPO:
    # the exact state stays in the chi = 2 manifold; serial 2TDVP converges
    # at second order, p2TDVP's retardation error vanishes as dt -> 0.
    L, T = 20, 1.0
    a, lam = [0.8, 0.2], [0.6, 0.3]
    Jr = lambda r: float(ti.expsum_J(a, lam, [r])[0])  # noqa: E731
    mps, c = ti.magnon_superposition_mps(L, 3)
    Hs, basis = D.magnon_hamiltonian(L, 1, Jr, 1.0)
    v = np.array([c[next(iter(b))] for b in basis])
    v = D.evolve(Hs, v / np.linalg.norm(v), T)
    ref = np.full(L, 0.5)
    for pb, b in zip(np.abs(v) ** 2, basis):
        ref[next(iter(b))] -= pb
    errs = []
    for dt in (0.1, 0.05):
        st = O.init_state(mps, ti.mpo_xxz_expsum(L, a, lam, 1.0), O.Params(chi_max=8), p)
        for _ in range(int(round(T / dt))):
            O.step(st, dt)
        errs.append(np.abs(O.measure(st)["sz"] - ref).max())
    if p == 1:
        assert errs[1] < 2e-5 and 3.5 < errs[0] / errs[1] < 4.5
    else:
        assert errs[1] < 0.6 * errs[0] and errs[1] < 5e-4


# --------------------------------------------------------------------------
# partition plan, directions, per-half counting (AMB-1 invariant)
# --------------------------------------------------------------------------

def test_partition_and_directions():
    assert O.plan_partition(128, 8) == [(16 * q, 16 * q + 15) for q in range(8)]
    assert O.plan_partition(129, 8)[0] == (0, 16)
    assert [e - s + 1 for s, e in O.plan_partition(131, 8)] == [18, 16, 16, 16, 16, 16, 16, 17]
    for bad in (3, 0, 7, 66):
        with pytest.raises(ValueError):
            O.plan_partition(128 if bad != 66 else 130, bad)
    assert O.directions(2, 1) == ["L", "R"]
    assert O.directions(4, 1) == ["R", "L", "R", "L"]
    assert O.directions(8, 1) == ["R", "L", "R", "L", "R", "L", "R", "L"]  # q=3 L, q=4 R
    assert O.directions(4, 2) == ["L", "R", "L", "R"]
    assert O.directions(1, 1) == ["R"] and O.directions(1, 2) == ["L"]


@pytest.mark.parametrize("L,p", [(8, 1), (8, 2), (12, 4), (16, 8), (10, 2)])
def test_counts_per_step(L, p):
    st = O.init_state(ti.neel_mps(L), ti.mpo_xxz_nn(L, 1.0), O.Params(chi_max=4), p)
    st.trace = True
    O.step(st, 0.05)
    pairs = [x for x in st.stats.log if x[0] == "pair"]
    full = [x for x in pairs if x[3] == -1.0j * 0.05]
    # N-1 forward pairs per half (merged counted twice), N-2 singles per half
    assert len(pairs) + len(full) == 2 * (L - 1)
    assert st.stats.n_back == 2 * (L - 2)
    # each bond gets total forward time dt: sum over pairs of |tau| per bond
    per_bond = np.zeros(L - 1)
    for _, q, j, tau in pairs:
        per_bond[j] += abs(tau)
    assert np.allclose(per_bond, 0.05)


def test_p13b_explicit_partition_converges_to_serial():
    """Any contiguous partition (here an uneven, load-balanced-style one) is a
    valid p2TDVP partition: its deviation from the serial run vanishes as
    dt -> 0 like the uniform one's (P13), and a malformed one is rejected."""
    L, T = 12, 0.4
    W = ti.mpo_xxz_nn(L, 0.5)
    bounds = [(0, 4), (5, 6), (7, 8), (9, 11)]
    devs = []
    for dt in (0.04, 0.02, 0.01):
        out = []
        for pp, bb in ((1, None), (4, bounds)):
            st = O.init_state(ti.neel_mps(L), W, O.Params(chi_max=64), pp, bb)
            assert [(s.s, s.e) for s in st.segs] == (bb or [(0, L - 1)])
            for _ in range(int(round(T / dt))):
                O.step(st, dt)
            out.append(O.measure(st)["sz"])
        devs.append(np.abs(out[0] - out[1]).max())
    assert devs[0] > devs[1] > devs[2]
    assert devs[2] < 1e-9
    for bad in ([(0, 4), (5, 11), (11, 11)], [(0, 5), (7, 11)], [(0, 0), (1, 11)], [(0, 3), (4, 7), (8, 11)]):
        with pytest.raises(ValueError):
            O.init_state(ti.neel_mps(L), W, O.Params(chi_max=64), len(bad), bad)
