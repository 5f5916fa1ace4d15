"""Plain CPU oracle of two-site DMRG on the 2TDVP data structures (SURVEY.md
§8(f) N3) -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper prepares every quench from a DMRG ground state ("ARPACK
... maximum of 8 basis vectors", :122, :130, :178 ground states of the Ising,
XY and XXX models).  Two-site DMRG is the same local step as the 2TDVP pair
update with the exponential replaced by the lowest eigenvector of H_eff^(2)
(PAPER.md:443-447 H_eff, :455 SVD split) and no one-site backward steps:

  sweep = left->right over pairs j = 0..L-2, then right->left over
          j = L-3..0 (the turnaround pair is optimised once per sweep)
  pair(j): Theta = Psi_j V_j Psi_{j+1};
           Theta' = lowest eigenvector of H_eff^(2) (restarted Lanczos below);
           SVD split and truncation exactly as svd_truncate (O-7);
           the environment for the next pair (beta_{j+1} sweeping right,
           gamma_j sweeping left; both at the two turnarounds).

Restarted Lanczos (a reading, DESIGN.md R-DMRG: the paper names ARPACK with 8
basis vectors and gives no restart rule): `restarts` times, build the K-vector
Lanczos basis from the current vector exactly as expm_lanczos (CGS2,
breakdown -> stop), take the lowest eigenpair (mu_0, y) of the tridiagonal
T = Q mu Q^T, normalise the sign so that y_0 >= 0 (the component along the
start vector), and restart from x = V y.  Returns (x, mu_0).
"""
from __future__ import annotations

import numpy as np

from .tdvp import (State, apply_h2, env_left, env_right, init_state, merge_theta, svd_truncate, _tridiag)


def lanczos_ground(apply, v, K=8, restarts=4, info=None):
    """Lowest eigenpair of a Hermitian operator by restarted Lanczos (see above)."""
    shape = v.shape
    x = v.reshape(-1).astype(np.complex128)
    x = x / np.linalg.norm(x)
    e0 = None
    for _ in range(restarts):
        V = [x]
        alpha, beta = [], []
        for k in range(K):
            w = apply(V[k].reshape(shape)).reshape(-1)
            a = float(np.real(np.vdot(V[k], w)))
            alpha.append(a)
            w = w - a * V[k]
            if k > 0:
                w = w - beta[k - 1] * V[k - 1]
            for _r in range(2):  # CGS2
                Vm = np.array(V)
                w = w - Vm.T @ (Vm.conj() @ w)
            b = float(np.linalg.norm(w))
            scale = max([1.0] + [abs(t) for t in alpha] + beta)
            if b <= 1e-12 * scale:
                break
            if k + 1 < K:
                beta.append(b)
                V.append(w / b)
        m = len(alpha)
        T = _tridiag(alpha, beta[: m - 1])
        mu, Q = np.linalg.eigh(T)
        y = Q[:, 0]
        if y[0] < 0:
            y = -y
        x = np.array(V[:m]).T @ y
        x = x / np.linalg.norm(x)
        e0 = float(mu[0])
    if info is not None:
        info["energy"] = e0
    return x.reshape(shape), e0


def _pair_ground(st: State, seg, j: int, restarts: int, build_beta: bool, build_gamma: bool):
    p = st.params
    th = merge_theta(seg.psi[j], 1.0 / seg.lam[j], seg.psi[j + 1])
    L_, R_ = seg.beta[j], seg.gamma[j + 1]
    W1, W2 = st.W[j], st.W[j + 1]
    th2, e0 = lanczos_ground(lambda x: apply_h2(L_, W1, W2, R_, x), th, p.krylov_k, restarts)
    if p.u1:
        from .u1 import svd_truncate_u1
        psi_l, S, psi_r, w, r, chi_eps, qm = svd_truncate_u1(th2, seg.qb[j], seg.qb[j + 2], p)
        seg.qb[j + 1] = qm
    else:
        psi_l, S, psi_r, w, r, chi_eps = svd_truncate(th2, p)
    seg.psi[j], seg.lam[j], seg.psi[j + 1] = psi_l, S, psi_r
    st.stats.w_step += w
    st.stats.n_pair += 1
    if len(S) < min(chi_eps, r):
        st.stats.trunc_active = True
    V = 1.0 / S
    if build_beta:
        seg.beta[j + 1] = env_left(seg.beta[j], psi_l * V[None, None, :], W1)
    if build_gamma:
        seg.gamma[j] = env_right(seg.gamma[j + 1], V[:, None, None] * psi_r, W2)
    return e0


def dmrg(mps, W, params, n_sweeps, restarts=4):
    """Two-site DMRG sweeps from the inverse-canonical `mps` (serial, one
    segment).  Returns (state, energies) with the Ritz value of the last pair
    update of every sweep."""
    st = init_state(mps, W, params, 1)
    seg = st.segs[0]
    L = st.L
    energies = []
    for _ in range(n_sweeps):
        st.stats.w_step = 0.0
        e = None
        for j in range(0, L - 1):  # left -> right
            e = _pair_ground(st, seg, j, restarts, True, j == L - 2)
        for j in range(L - 3, -1, -1):  # right -> left
            e = _pair_ground(st, seg, j, restarts, j == 0, True)
        energies.append(e)
    return st, energies
