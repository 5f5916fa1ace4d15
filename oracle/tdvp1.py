"""Plain CPU oracle of serial one-site TDVP (1TDVP) and the hybrid 2TDVP -> 1TDVP
scheme (arXiv:1912.06127).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  complex128 throughout.

PAPER.md:697 (§V): "a parallel variant of one-site TDVP (p1TDVP) ... would
enable a parallel version of the hybrid method ..., whereby a simulation
starts with 2TDVP and switches to 1TDVP when chi_max is saturated.  1TDVP is
faster".  The paper gives no p1TDVP algorithm; what is built here is the
serial one-site integrator the hybrid switches to, in the paper's own
building blocks and storage (reading R-1TDVP in DESIGN.md), and its
segment-parallel form (step1p, reading R-P1TDVP, below):

* the state is kept in the inverse-canonical product form
  Psi_0 V_0 Psi_1 ... Psi_{L-1}, every bond split by the
  same truncated SVD as the 2TDVP pair update (O-7);
* a forward one-site step is exp(-i tau H_eff^(1)) on a site (the 2TDVP
  backward step with the opposite sign);
* a backward bond ("zero-site") step is exp(+i tau H_eff^(0)) on the bond
  matrix C, with H_eff^(0) C [a, b] = sum L[a, w, a'] R[b, w, b'] C[a', b']
  (the one-site Fig 5b contraction without a site tensor);
* one step = left-to-right sweep then right-to-left sweep, tau = dt/2 each,
  the two consecutive forward steps of the last site merged into one of dt
  (the turnaround merge of PAPER.md:430, exact: the same H_eff^(1)).

Right sweep, site j (centre Psi_j; bond j to its right):
  Psi_j <- exp(-i tau H1(beta_j, W_j, gamma_j)) Psi_j   (tau = dt at j = L-1)
  B = diag(V_j) Psi_{j+1}                                 (right-canonical)
  Psi_j (cl d x cr) = U S W^dag (truncated SVD, O-7):  Psi_j = U S, V_j = 1/S
  beta_{j+1} = env_left(beta_j, U, W_j)
  C = S W^dag;  C <- exp(+i tau H0(beta_{j+1}, gamma_j)) C
  Psi_{j+1} = C B
Left sweep, site j (mirror; the last site was already evolved by dt):
  Psi_j <- exp(-i tau H1) Psi_j                           (j < L-1)
  A = Psi_{j-1} diag(V_{j-1})                             (left-canonical)
  Psi_j (cl x d cr) = U S W^dag:  Psi_j = S W^dag, V_{j-1} = 1/S
  gamma_{j-1} = env_right(gamma_j, W^dag, W_j)
  C = U S;  C <- exp(+i tau H0(beta_j, gamma_{j-1})) C
  Psi_{j-1} = A C
"""
from __future__ import annotations

import numpy as np

from .tdvp import (Params, State, apply_h1, env_left, env_right, expm_lanczos, svd_truncate)


def apply_h0(L, R, C):
    """H_eff^(0) C (bond matrix): out[a, b] = sum L[a, w, a'] R[b, w, b'] C[a', b']."""
    T = np.tensordot(L, C, axes=(2, 0))                   # [a, w, b']
    return np.tensordot(T, R, axes=([1, 2], [1, 2]))      # [a, b]


def _split(M, p: Params):
    """Truncated SVD of a matrix M (m x n) by the 2TDVP rule (O-7):
    (U S (m x chi), S, S W^dag (chi x n), discarded weight)."""
    m, n = M.shape
    psi_l, S, psi_r, w, _, _ = svd_truncate(M.reshape(m, 1, 1, n), p)
    return psi_l.reshape(m, -1), S, psi_r.reshape(-1, n), w


def step1(st: State, dt: float):
    """One serial 1TDVP step on a p = 1 State (see the module docstring)."""
    if st.p != 1:
        raise ValueError("1TDVP is serial (p = 1)")
    seg = st.segs[0]
    p = st.params
    L = st.L
    W = st.W
    tau = 0.5 * dt
    st.stats.w_step = 0.0
    info = {}

    def fwd(j, t):
        seg.psi[j] = expm_lanczos(lambda x: apply_h1(seg.beta[j], W[j], seg.gamma[j], x), seg.psi[j], -1j * t,
                                  p.krylov_k, p.krylov_tol, info)
        st.stats.krylov_breakdowns += int(info.get("breakdown", False))

    def bwd_bond(Lenv, Renv, C):
        out = expm_lanczos(lambda x: apply_h0(Lenv, Renv, x), C, 1j * tau, p.krylov_k, p.krylov_tol, info)
        st.stats.krylov_breakdowns += int(info.get("breakdown", False))
        return out

    # left-to-right
    for j in range(L):
        fwd(j, dt if j == L - 1 else tau)
        if j == L - 1:
            break
        cl, d, cr = seg.psi[j].shape
        B = (1.0 / seg.lam[j])[:, None, None] * seg.psi[j + 1]
        US, S, SWh, w = _split(seg.psi[j].reshape(cl * d, cr), p)
        st.stats.w_step += w
        chi = len(S)
        seg.psi[j] = US.reshape(cl, d, chi)
        seg.lam[j] = S
        U = seg.psi[j] * (1.0 / S)[None, None, :]
        seg.beta[j + 1] = env_left(seg.beta[j], U, W[j])
        C = bwd_bond(seg.beta[j + 1], seg.gamma[j], SWh)
        seg.psi[j + 1] = np.tensordot(C, B, axes=(1, 0))
    # right-to-left
    for j in range(L - 1, -1, -1):
        if j < L - 1:
            fwd(j, tau)
        if j == 0:
            break
        cl, d, cr = seg.psi[j].shape
        A = seg.psi[j - 1] * (1.0 / seg.lam[j - 1])[None, None, :]
        US, S, SWh, w = _split(seg.psi[j].reshape(cl, d * cr), p)
        st.stats.w_step += w
        chi = len(S)
        seg.psi[j] = SWh.reshape(chi, d, cr)
        seg.lam[j - 1] = S
        Wh = (1.0 / S)[:, None, None] * seg.psi[j]
        seg.gamma[j - 1] = env_right(seg.gamma[j], Wh, W[j])
        C = bwd_bond(seg.beta[j], seg.gamma[j - 1], US)
        seg.psi[j - 1] = np.tensordot(A, C, axes=(2, 0))
    st.stats.w_total += st.stats.w_step


# ----------------------------------------------------------------------------
# segment-parallel one-site TDVP (p1TDVP, reading R-P1TDVP in DESIGN.md)
# ----------------------------------------------------------------------------
#
# PAPER.md:697 expects "a parallel variant of one-site TDVP (p1TDVP) could be
# developed using the same approach" as p2TDVP.  Reading: the App. A half-step
# programs unchanged at the segment boundaries -- D and C phases keep the
# paper's two-site Lambda^-1-merged boundary pair updates, the
# D-phase backward one-site step and the half-1/half-2 merge of full-dt
# boundary pairs -- and every segment's interior sweep one-site:
#   RIGHT over [s, e]: [back(s) if q > 0]; site_right(j) for j = s .. e-1
#     (forward Psi_j by dt/2 unless merged, split bond j, beta_{j+1}, backward
#     bond j by dt/2, absorb into Psi_{j+1}); at the chain end e = L-1 the last
#     site forward by dt in half 1 (merged: skipped in half 2), dt/2 in half 2
#   LEFT over [s, e]: [back(e) if q < p-1]; site_left(j) for j = e .. s+1
#     (mirror: split bond j-1, gamma_{j-1}, absorb into Psi_{j-1}); at the
#     chain start s = 0 site 0 forward by dt in half 1, dt/2 in half 2.
# Per step every site is evolved forward by dt and every interior bond
# backward by dt, as in serial 1TDVP; every boundary as in p2TDVP.  p = 1 is
# exactly step1.


def _fwd(st, seg, j, t):
    p = st.params
    info = {}
    seg.psi[j] = expm_lanczos(lambda x: apply_h1(seg.beta[j], st.W[j], seg.gamma[j], x), seg.psi[j], -1j * t,
                              p.krylov_k, p.krylov_tol, info)
    st.stats.krylov_breakdowns += int(info.get("breakdown", False))


def _bond_back(st, Lenv, Renv, C, tau):
    p = st.params
    info = {}
    out = expm_lanczos(lambda x: apply_h0(Lenv, Renv, x), C, 1j * tau, p.krylov_k, p.krylov_tol, info)
    st.stats.krylov_breakdowns += int(info.get("breakdown", False))
    return out


def _site_right(st, seg, j, t_fwd, tau):
    """Forward site j by t_fwd (None: already evolved), split bond j, beta_{j+1},
    bond j backward by tau, absorb into site j+1."""
    if t_fwd is not None:
        _fwd(st, seg, j, t_fwd)
    cl, d, cr = seg.psi[j].shape
    B = (1.0 / seg.lam[j])[:, None, None] * seg.psi[j + 1]
    US, S, SWh, w = _split(seg.psi[j].reshape(cl * d, cr), st.params)
    st.stats.w_step += w
    seg.psi[j] = US.reshape(cl, d, len(S))
    seg.lam[j] = S
    seg.beta[j + 1] = env_left(seg.beta[j], seg.psi[j] * (1.0 / S)[None, None, :], st.W[j])
    C = _bond_back(st, seg.beta[j + 1], seg.gamma[j], SWh, tau)
    seg.psi[j + 1] = np.tensordot(C, B, axes=(1, 0))


def _site_left(st, seg, j, t_fwd, tau):
    """Forward site j by t_fwd (None: already evolved), split bond j-1,
    gamma_{j-1}, bond j-1 backward by tau, absorb into site j-1."""
    if t_fwd is not None:
        _fwd(st, seg, j, t_fwd)
    cl, d, cr = seg.psi[j].shape
    A = seg.psi[j - 1] * (1.0 / seg.lam[j - 1])[None, None, :]
    US, S, SWh, w = _split(seg.psi[j].reshape(cl, d * cr), st.params)
    st.stats.w_step += w
    seg.psi[j] = SWh.reshape(len(S), d, cr)
    seg.lam[j - 1] = S
    seg.gamma[j - 1] = env_right(seg.gamma[j], (1.0 / S)[:, None, None] * seg.psi[j], st.W[j])
    C = _bond_back(st, seg.beta[j], seg.gamma[j - 1], US, tau)
    seg.psi[j - 1] = np.tensordot(A, C, axes=(2, 0))


def _half1(st: State, dt: float, h: int, merged_pairs: set, merged_sites: set):
    """Half h of a p1TDVP step, phase by phase (the structure of tdvp._half)."""
    from .tdvp import LEFT, RIGHT, _back, _pair, directions
    L, p = st.L, st.p
    dirs = directions(p, h)
    th, tf = 0.5 * dt, dt
    tau_h, tau_f = -0.5j * dt, -1.0j * dt
    new_pairs, new_sites = set(), set()
    # ---- D-phase: unchanged two-site boundary updates
    for q in range(p - 1):
        if dirs[q] == LEFT and dirs[q + 1] == RIGHT:
            a, b = st.segs[q], st.segs[q + 1]
            e = a.e
            if e not in merged_pairs:
                _pair(st, a, e, tau_h, True, True)
                b.psi[e + 1] = a.psi[e + 1].copy()
                b.lam[e] = a.lam[e].copy()
                b.beta[e + 1] = a.beta[e + 1].copy()
    # ---- sweep phase: one-site interiors
    for seg in st.segs:
        q, s, e = seg.q, seg.s, seg.e
        if dirs[q] == RIGHT:
            if q > 0:
                _back(st, seg, s, dt)
            for j in range(s, e):
                _site_right(st, seg, j, None if j in merged_sites else th, th)
            if e == L - 1 and (L - 1) not in merged_sites:
                _fwd(st, seg, L - 1, tf if h == 1 else th)
                if h == 1:
                    new_sites.add(L - 1)
        else:
            if q < p - 1:
                _back(st, seg, e, dt)
            for j in range(e, s, -1):
                _site_left(st, seg, j, None if j in merged_sites else th, th)
            if s == 0 and 0 not in merged_sites:
                _fwd(st, seg, 0, tf if h == 1 else th)
                if h == 1:
                    new_sites.add(0)
    # ---- C-phase: unchanged two-site boundary updates
    for q in range(p - 1):
        if dirs[q] == RIGHT and dirs[q + 1] == LEFT:
            a, b = st.segs[q], st.segs[q + 1]
            e, s = a.e, b.s
            a.psi[s] = b.psi[s].copy()
            a.gamma[s] = b.gamma[s].copy()
            tau = tau_f if h == 1 else tau_h
            _pair(st, a, e, tau, True, True)
            if tau == tau_f:
                new_pairs.add(e)
            b.psi[s] = a.psi[s].copy()
            b.lam[e] = a.lam[e].copy()
            b.beta[s] = a.beta[s].copy()
    return new_pairs, new_sites


def step1p(st: State, dt: float):
    """One p1TDVP step (half 1 + half 2) on a State of any p (reading above);
    p = 1 is step1."""
    if st.params.u1:
        raise ValueError("p1TDVP runs in dense mode")
    st.stats.w_step = 0.0
    st.stats.trunc_active = False
    mp, ms = _half1(st, dt, 1, set(), set())
    _half1(st, dt, 2, mp, ms)
    st.stats.w_total += st.stats.w_step


def saturated(chi, L: int, d: int, chi_max: int) -> bool:
    """Hybrid switch rule ("switches to 1TDVP when chi_max is
    saturated"): every bond at its largest possible dimension
    min(chi_max, d^(j+1), d^(L-j-1)) (SURVEY.md §8(d) bond bound).  chi is the
    (L+1)-entry profile with chi[0] = chi[L] = 1."""
    for j in range(L - 1):
        cap = min(chi_max, d ** min(j + 1, L - j - 1))
        if chi[j + 1] < cap:
            return False
    return True


def step_hybrid(st: State, dt: float, d: int = 2) -> int:
    """One step of the hybrid scheme: (p)2TDVP until chi_max is saturated on
    every bond, then (p)1TDVP on the same partition (R-P1TDVP).  Returns 1 or
    2 (the integrator used)."""
    from .tdvp import chi_profile, step
    if saturated(chi_profile(st), st.L, d, st.params.chi_max):
        step1p(st, dt)
        return 1
    step(st, dt)
    return 2
