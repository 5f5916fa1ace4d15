"""Plain CPU oracle of serial 2TDVP and p2TDVP (arXiv:1912.06127).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  complex128 throughout.
Every function cites the PAPER.md passage it follows; readings of silent or
garbled passages are the SURVEY.md §8(c) "AMB-n" readings, listed in
DESIGN.md.  Index conventions:

  Psi_j  (chi_l, d, chi_r)      Lambda_j, V_j = 1/Lambda_j  float64 (chi_j,)
  W_j    (D_l, d_out, d_in, D_r) with W[w, s, t, w'] = <s|O|t>
  beta_j, gamma_j  (chi, D, chi): first index bra (conjugated), last ket
  theta  (chi_L, d, d, chi_R)

Contractions are np.tensordot steps in the order the index formula is
written; nothing is blocked, fused or reordered beyond pairwise contraction.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

# ----------------------------------------------------------------------------
# parameters
# ----------------------------------------------------------------------------


@dataclass
class Params:
    """Truncation/Krylov knobs (PAPER.md:100 S-IV defaults)."""

    chi_max: int
    eps: float = 1e-12          # relative SV cutoff epsilon
    w_max: float = 0.0          # per-SVD discarded-weight tolerance; 0 = off
    krylov_k: int = 8           # max Krylov vectors
    krylov_tol: float = 0.0     # 0 = always K vectors (parity mode, AMB-5)
    multiplet_delta: float = 1e-6  # AMB-9 multiplet guard
    u1: bool = False            # S^z-conserving block-sparse SVD (oracle/u1.py)


# ----------------------------------------------------------------------------
# local contractions
# ----------------------------------------------------------------------------


def env_left(beta, A, W):
    """beta'[b,w',b'] = sum conj(A[a,s,b]) beta[a,w,a'] W[w,s,t,w'] A[a',t,b'].

    PAPER.md:447-451 (§III.A): "a new lefthand environment beta_{j+1} is
    created from the contraction of beta_j, Psi_j, V_j, Psi_j^dagger, V_j and
    the Hamiltonian MPO tensor"; the caller passes A = Psi_j diag(V_j).
    """
    X = np.tensordot(beta, A, axes=(2, 0))             # [a, w, t, b']
    Y = np.tensordot(X, W, axes=([1, 2], [0, 2]))       # [a, b', s, w']
    out = np.tensordot(A.conj(), Y, axes=([0, 1], [0, 2]))  # [b, b', w']
    return np.ascontiguousarray(out.transpose(0, 2, 1))


def env_right(gamma, B, W):
    """gamma'[a,w,a'] = sum conj(B[a,s,b]) W[w,s,t,w'] B[a',t,b'] gamma[b,w',b'].

    Mirror of env_left (PAPER.md:427 Fig 3b, :432); B = diag(V_{j-1}) Psi_j.
    """
    X = np.tensordot(B, gamma, axes=(2, 2))             # [a', t, b, w']
    Y = np.tensordot(X, W, axes=([1, 3], [2, 3]))       # [a', b, w, s]
    out = np.tensordot(B.conj(), Y, axes=([1, 2], [3, 1]))  # [a, a', w]
    return np.ascontiguousarray(out.transpose(0, 2, 1))


def apply_h2(L, W1, W2, R, theta):
    """H_eff^(2) theta (Fig 5a; never formed explicitly).

    out[a,s1,s2,b] = sum L[a,w,a'] W1[w,s1,t1,w'] W2[w',s2,t2,w''] R[b,w'',b'] theta[a',t1,t2,b']
    """
    T1 = np.tensordot(L, theta, axes=(2, 0))            # [a, w, t1, t2, b']
    T2 = np.tensordot(T1, W1, axes=([1, 2], [0, 2]))    # [a, t2, b', s1, w']
    T3 = np.tensordot(T2, W2, axes=([1, 4], [2, 0]))    # [a, b', s1, s2, w'']
    return np.tensordot(T3, R, axes=([1, 4], [2, 1]))   # [a, s1, s2, b]


def apply_h1(L, W, R, psi):
    """H_eff^(1) psi (Fig 5b).

    out[a,s,b] = sum L[a,w,a'] W[w,s,t,w'] R[b,w',b'] psi[a',t,b']
    """
    T1 = np.tensordot(L, psi, axes=(2, 0))              # [a, w, t, b']
    T2 = np.tensordot(T1, W, axes=([1, 2], [0, 2]))     # [a, b', s, w']
    return np.tensordot(T2, R, axes=([1, 3], [2, 1]))   # [a, s, b]


def merge_theta(psi_l, v, psi_r):
    """Theta[a,s1,s2,b] = sum_k Psi_j[a,s1,k] V_j[k] Psi_{j+1}[k,s2,b].

    Inverse-canonical two-site state (Fig 5a).
    """
    return np.tensordot(psi_l * v[None, None, :], psi_r, axes=(2, 0))


MULTIPLET_ABS = 1e-13  # absolute degeneracy floor of the multiplet guard (reading R-9b)

# ----------------------------------------------------------------------------
# truncated SVD (PAPER.md:455 Fig 6; :493-499 eq:discweight; :510 epsilon)
# ----------------------------------------------------------------------------


def truncation_rank(sigma, p: Params):
    """Kept rank chi for descending singular values sigma.

    chi_eps = #{sigma_k >= eps sigma_1}
    chi_w   = min chi with sum_{k>chi} sigma_k^2 <= w_max
              (w_max = 0 -> chi_w = #nonzero)
    chi     = min(chi_eps, chi_w, chi_max), then the multiplet guard:
              while 1 < chi < r and sigma_chi - sigma_{chi+1} <= delta sigma_chi + tau sigma_1:
                  chi -= 1
              with tau = MULTIPLET_ABS = 1e-13: values closer than the absolute accuracy of
              any backward-stable SVD (O(u sigma_1)) are one multiplet, so a
              numerically degenerate multiplet (e.g. SU(2) at Delta = 1) straddling
              the eps cut is kept or dropped whole (reading R-9b).
    eps = 0 is floored at 1e-14 (SPEC.md linalg-core design decision) so that
    V = 1/Lambda never overflows (PAPER.md:365 footnote).
    """
    r = len(sigma)
    s1 = sigma[0]
    eps = p.eps if p.eps > 0 else 1e-14
    chi_eps = int(np.count_nonzero(sigma >= eps * s1))
    nz = int(np.count_nonzero(sigma > 0))
    if p.w_max > 0:
        sq = sigma.astype(np.float64) ** 2
        chi_w = nz
        # tail[c] = sum_{k >= c} sigma_k^2 (0-based): weight discarded keeping c
        tail = np.concatenate([np.cumsum(sq[::-1])[::-1], [0.0]])
        for c in range(0, r + 1):
            if tail[c] <= p.w_max:
                chi_w = c
                break
        chi_w = max(chi_w, 1)
    else:
        chi_w = nz
    chi = max(1, min(chi_eps, chi_w, p.chi_max))
    while 1 < chi < r and sigma[chi - 1] - sigma[chi] <= p.multiplet_delta * sigma[chi - 1] + MULTIPLET_ABS * s1:
        chi -= 1
    return chi


def svd_truncate(theta, p: Params):
    """Split Theta' = A' Lambda' B' (Fig 6), truncated (O-7).

    Reshape rows (a, s1), cols (s2, b) (AMB-17).  Returns
    (Psi_L' = A' Lambda', Lambda', Psi_R' = Lambda' B', w, chi_full, chi_eps)
    with w = sum_{k > chi} sigma_k^2 (eq:discweight, absolute).
    """
    cl, d1, d2, cr = theta.shape
    M = theta.reshape(cl * d1, d2 * cr)
    if not np.all(np.isfinite(M)):
        raise FloatingPointError("non-finite Theta before SVD")
    u, s, vh = scipy.linalg.svd(M, full_matrices=False, lapack_driver="gesvd")
    if s[0] <= 0:
        raise FloatingPointError("all singular values zero")
    chi = truncation_rank(s, p)
    w = float(np.sum(s[chi:] ** 2))
    S = s[:chi].copy()
    psi_l = (u[:, :chi] * S[None, :]).reshape(cl, d1, chi)
    psi_r = (S[:, None] * vh[:chi]).reshape(chi, d2, cr)
    eps = p.eps if p.eps > 0 else 1e-14
    chi_eps = int(np.count_nonzero(s >= eps * s[0]))
    return psi_l, S, psi_r, w, len(s), chi_eps


# ----------------------------------------------------------------------------
# Lanczos exponentiation (PAPER.md:447 + footnote; :100 "max 8 vectors")
# ----------------------------------------------------------------------------


def expm_lanczos(apply, v, tau, K=8, tol=0.0, info=None):
    """exp(tau H) v from a Lanczos basis of at most K vectors.

    1. n0 = ||v||, v_1 = v / n0
    2. for k = 1..K: w = H v_k; alpha_k = Re<v_k, w>;
       w -= alpha_k v_k + beta_{k-1} v_{k-1}; two classical Gram-Schmidt
       passes against v_1..v_k; beta_k = ||w||;
       breakdown if beta_k <= 1e-12 * max(1, |alpha_1..k|, beta_1..k-1)
    3. T = tridiag(alpha, beta) = Q mu Q^T (real symmetric)
    4. result = n0 V (Q (e^{tau mu} * Q^T e_1))
    tol > 0: stop early once n0 beta_k |c_k| < tol (paper mode); tol = 0: K.
    """
    shape = v.shape
    x = v.reshape(-1).astype(np.complex128)
    n0 = float(np.linalg.norm(x))
    if n0 == 0.0:
        return v.copy()
    V = [x / n0]
    alpha, beta = [], []
    breakdown = False
    for k in range(K):
        w = apply(V[k].reshape(shape)).reshape(-1)
        a = float(np.real(np.vdot(V[k], w)))
        alpha.append(a)
        w = w - a * V[k]
        if k > 0:
            w = w - beta[k - 1] * V[k - 1]
        for _ in range(2):  # CGS2 full reorthogonalisation
            Vm = np.array(V)
            w = w - Vm.T @ (Vm.conj() @ w)
        b = float(np.linalg.norm(w))
        scale = max([1.0] + [abs(t) for t in alpha] + beta)
        if b <= 1e-12 * scale:
            breakdown = True
            break
        if tol > 0.0:
            Tk = _tridiag(alpha, beta)
            mu, Q = np.linalg.eigh(Tk)
            c = Q @ (np.exp(tau * mu) * Q[0, :])
            if n0 * b * abs(c[-1]) < tol:
                break
        beta.append(b)
        if k + 1 < K:
            V.append(w / b)
    m = len(alpha)
    T = _tridiag(alpha, beta[: m - 1])
    mu, Q = np.linalg.eigh(T)
    c = Q @ (np.exp(tau * mu) * Q[0, :])
    out = n0 * (np.array(V[:m]).T @ c)
    if info is not None:
        info["k"] = m
        info["breakdown"] = breakdown
    return out.reshape(shape)


def _tridiag(alpha, beta):
    m = len(alpha)
    T = np.diag(np.array(alpha, dtype=np.float64))
    for i in range(m - 1):
        T[i, i + 1] = T[i + 1, i] = beta[i]
    return T


# ----------------------------------------------------------------------------
# partitioning and sweep directions (§III.B, Fig 7)
# ----------------------------------------------------------------------------


def plan_partition(L: int, p: int):
    """Contiguous segments [(s, e)].

    p = 1 or p even with 2 <= p <= L/2, each segment >= 2 sites
    ("a partition must contain a minimum of two site tensors").
    Remainder sites go one at a time to segment 0, then p-1, then 0, ...
    """
    if p != 1 and (p % 2 != 0 or p < 2 or p > L // 2):
        raise ValueError(f"invalid number of segments p={p} for L={L}")
    base, rem = divmod(L, p)
    sizes = [base] * p
    i = 0
    while rem > 0:
        sizes[0 if i % 2 == 0 else p - 1] += 1
        rem -= 1
        i += 1
    segs, s = [], 0
    for n in sizes:
        segs.append((s, s + n - 1))
        s += n
    if p > 1 and min(sizes) < 2:
        raise ValueError("segment shorter than two sites")
    return segs


def check_partition(L: int, bounds):
    """Validate explicit segment bounds [(s, e)]: contiguous from 0 to L-1,
    p = 1 or p even (the direction rule of PAPER.md:470 pairs segments), every
    segment >= 2 sites when p > 1.  Returns them as tuples."""
    b = [(int(s), int(e)) for s, e in bounds]
    p = len(b)
    if p != 1 and (p % 2 != 0 or p < 2):
        raise ValueError(f"invalid number of segments p={p}")
    if b[0][0] != 0 or b[-1][1] != L - 1 or any(b[q + 1][0] != b[q][1] + 1 for q in range(p - 1)):
        raise ValueError("segments must be contiguous and cover 0..L-1")
    if p > 1 and min(e - s + 1 for s, e in b) < 2:
        raise ValueError("segment shorter than two sites")
    return b


RIGHT, LEFT = "R", "L"


def directions(p: int, h: int):
    """Sweep direction of each segment in half h.

    Half 1: q sweeps LEFT iff q = p/2 - 1 (mod 2), so the two central
    segments sweep away from the centre and neighbours alternate; half 2
    reverses all.  p = 1: RIGHT then LEFT.
    """
    if p == 1:
        d = [RIGHT]
    else:
        d = [LEFT if (q % 2) == ((p // 2 - 1) % 2) else RIGHT for q in range(p)]
    if h == 2:
        d = [LEFT if x == RIGHT else RIGHT for x in d]
    return d


# ----------------------------------------------------------------------------
# state: one "world" per segment (message passing between neighbours)
# ----------------------------------------------------------------------------


class Segment:
    """Everything one process owns.

    psi: sites s..e plus the right ghost e+1 (the neighbour's Psi, held for
    boundary updates); lam: bonds it owns (s..e, boundary bond e owned by
    the left process, AMB-4) plus the received Lambda_{s-1};
    beta/gamma: envs of sites s..e+1.
    """

    def __init__(self, q, s, e):
        self.q, self.s, self.e = q, s, e
        self.psi, self.lam, self.beta, self.gamma = {}, {}, {}, {}
        self.qb = {}  # U(1) mode: bond charges by bond position k (bond left of site k)


@dataclass
class Stats:
    w_step: float = 0.0
    w_total: float = 0.0
    trunc_active: bool = False
    n_svd: int = 0
    n_pair: int = 0
    n_back: int = 0
    krylov_breakdowns: int = 0
    log: list = field(default_factory=list)  # optional op trace


class State:
    def __init__(self, W, params: Params, p: int, bounds=None):
        self.W = [np.asarray(w, dtype=np.complex128) for w in W]
        self.L = len(W)
        self.params = params
        self.p = p
        # explicit bounds (any contiguous partition, e.g. load-balanced) or the uniform rule O-3
        self.bounds = plan_partition(self.L, p) if bounds is None else check_partition(self.L, bounds)
        if len(self.bounds) != p:
            raise ValueError("len(bounds) != p")
        self.segs = [Segment(q, s, e) for q, (s, e) in enumerate(self.bounds)]
        self.stats = Stats()
        self.trace = False


def _mps_envs(psi, lam, W):
    """All beta_j (L->R) and gamma_j (R->L) of a global inverse-canonical MPS.

    O-2: beta_0 = gamma_{L-1} = [[[1]]];
    beta_{j+1} = env_left(beta_j, Psi_j diag(V_j), W_j);
    gamma_{j-1} = env_right(gamma_j, diag(V_{j-1}) Psi_j, W_j).
    """
    L = len(psi)
    one = np.ones((1, 1, 1), dtype=np.complex128)
    beta = [None] * L
    gamma = [None] * L
    beta[0] = one
    for j in range(L - 1):
        beta[j + 1] = env_left(beta[j], psi[j] * (1.0 / lam[j])[None, None, :], W[j])
    gamma[L - 1] = one
    for j in range(L - 1, 0, -1):
        gamma[j - 1] = env_right(gamma[j], (1.0 / lam[j - 1])[:, None, None] * psi[j], W[j])
    return beta, gamma


def init_state(mps, W, params: Params, p: int = 1, bounds=None) -> State:
    """Sequential initial environments, handed to each segment's owner (O-2).
    `bounds`: explicit segment bounds [(s, e)] instead of the uniform rule."""
    st = State(W, params, p, bounds)
    L = st.L
    psi = [np.asarray(x, dtype=np.complex128) for x in mps.psi]
    lam = [np.asarray(x, dtype=np.float64) for x in mps.lam]
    if len(psi) != L:
        raise ValueError("MPS and MPO lengths differ")
    for l in lam:
        if np.any(l <= 0) or not np.all(np.isfinite(l)):
            raise ValueError("Lambda must be finite and > 0")
    beta, gamma = _mps_envs(psi, lam, st.W)
    qb = None
    if params.u1:
        from .u1 import infer_charges
        qb = infer_charges(psi)
    for seg in st.segs:
        if qb is not None:
            seg.qb = {k: qb[k].copy() for k in range(L + 1)}
        hi = min(seg.e + 1, L - 1)
        for j in range(seg.s, hi + 1):
            seg.psi[j] = psi[j].copy()
            seg.beta[j] = beta[j].copy()
            seg.gamma[j] = gamma[j].copy()
        for b in range(max(seg.s - 1, 0), min(seg.e, L - 2) + 1):
            seg.lam[b] = lam[b].copy()
    return st


# ----------------------------------------------------------------------------
# local updates
# ----------------------------------------------------------------------------


def _pair(st: State, seg: Segment, j: int, tau: complex, build_beta: bool, build_gamma: bool):
    """Two-site forward update of (j, j+1) on seg.

    Theta = Psi_j V_j Psi_{j+1}; Theta' = exp(tau H_eff^(2)) Theta
    (PAPER.md:443-447); SVD split Psi_j = U S, V_j = 1/S, Psi_{j+1} = S W^dagger
    (PAPER.md:455); then the env(s) needed next.
    """
    p = st.params
    th = merge_theta(seg.psi[j], 1.0 / seg.lam[j], seg.psi[j + 1])
    L_, R_ = seg.beta[j], seg.gamma[j + 1]
    W1, W2 = st.W[j], st.W[j + 1]
    info = {}
    th2 = expm_lanczos(lambda x: apply_h2(L_, W1, W2, R_, x), th, tau,
                       p.krylov_k, p.krylov_tol, info)
    st.stats.krylov_breakdowns += int(info.get("breakdown", False))
    if p.u1:
        from .u1 import svd_truncate_u1
        psi_l, S, psi_r, w, r, chi_eps, qm = svd_truncate_u1(th2, seg.qb[j], seg.qb[j + 2], p)
        seg.qb[j + 1] = qm
    else:
        psi_l, S, psi_r, w, r, chi_eps = svd_truncate(th2, p)
    seg.psi[j], seg.lam[j], seg.psi[j + 1] = psi_l, S, psi_r
    st.stats.w_step += w
    st.stats.n_svd += 1
    st.stats.n_pair += 1
    if len(S) < min(chi_eps, r):
        st.stats.trunc_active = True
    V = 1.0 / S
    if build_beta:
        seg.beta[j + 1] = env_left(seg.beta[j], psi_l * V[None, None, :], W1)
    if build_gamma:
        seg.gamma[j] = env_right(seg.gamma[j + 1], V[:, None, None] * psi_r, W2)
    if st.trace:
        st.stats.log.append(("pair", seg.q, j, tau))


def _back(st: State, seg: Segment, j: int, dt: float):
    """One-site backward update Psi_j <- exp(+i dt/2 H_eff^(1)) Psi_j."""
    p = st.params
    L_, R_, W = seg.beta[j], seg.gamma[j], st.W[j]
    info = {}
    seg.psi[j] = expm_lanczos(lambda x: apply_h1(L_, W, R_, x), seg.psi[j], 0.5j * dt,
                              p.krylov_k, p.krylov_tol, info)
    st.stats.krylov_breakdowns += int(info.get("breakdown", False))
    st.stats.n_back += 1
    if st.trace:
        st.stats.log.append(("back", seg.q, j))


# ----------------------------------------------------------------------------
# one half-step: D-phase -> sweep phase -> C-phase
# ----------------------------------------------------------------------------


def _half(st: State, dt: float, h: int, merged: set):
    """Execute half h of a p2TDVP step sequentially, phase by phase.

    Between the D and C phases segments are independent, so running every
    segment's D-part, then every sweep, then every C-part gives exactly the
    message-passing result (SURVEY.md App. A "Independence").
    Returns the set of pairs evolved with the full step (O-9 turnaround).
    """
    L, p = st.L, st.p
    dirs = directions(p, h)
    tau_h, tau_f = -0.5j * dt, -1.0j * dt
    new_merged = set()

    # ---- D-phase: left process of each diverging boundary updates the pair
    # ("we let the lefthand process update the boundary sites")
    for q in range(p - 1):
        if dirs[q] == LEFT and dirs[q + 1] == RIGHT:
            a, b = st.segs[q], st.segs[q + 1]
            e = a.e
            if e not in merged:
                _pair(st, a, e, tau_h, True, True)
                # send Psi'_{e+1}, Lambda'_e, beta_{e+1} to q+1
                b.psi[e + 1] = a.psi[e + 1].copy()
                b.lam[e] = a.lam[e].copy()
                b.beta[e + 1] = a.beta[e + 1].copy()
                if st.params.u1:
                    b.qb[e + 1] = a.qb[e + 1].copy()

    # ---- sweep phase
    for seg in st.segs:
        q, s, e = seg.q, seg.s, seg.e
        if dirs[q] == RIGHT:
            if q > 0:
                _back(st, seg, s, dt)
            for j in range(s, e):
                if j not in merged:
                    tau = tau_f if (h == 1 and j + 1 == L - 1) else tau_h
                    full = tau == tau_f
                    _pair(st, seg, j, tau, not full, full)
                    if full:
                        new_merged.add(j)
                if not (j + 1 == e and e == L - 1):
                    _back(st, seg, j + 1, dt)
        else:
            if q < p - 1:
                _back(st, seg, e, dt)
            for j in range(e - 1, s - 1, -1):
                if j not in merged:
                    tau = tau_f if (h == 1 and j == 0) else tau_h
                    full = tau == tau_f
                    _pair(st, seg, j, tau, full, not full)
                    if full:
                        new_merged.add(j)
                if not (j == s and s == 0):
                    _back(st, seg, j, dt)

    # ---- C-phase: converging boundaries
    for q in range(p - 1):
        if dirs[q] == RIGHT and dirs[q + 1] == LEFT:
            a, b = st.segs[q], st.segs[q + 1]
            e = a.e
            s = b.s
            # right sends Psi_s, gamma_s to left
            a.psi[s] = b.psi[s].copy()
            a.gamma[s] = b.gamma[s].copy()
            if st.params.u1:
                a.qb[s + 1] = b.qb[s + 1].copy()
            tau = tau_f if h == 1 else tau_h
            _pair(st, a, e, tau, True, True)
            if tau == tau_f:
                new_merged.add(e)
            # left sends Psi'_{e+1}, Lambda'_e, beta_{e+1} back
            b.psi[s] = a.psi[s].copy()
            b.lam[e] = a.lam[e].copy()
            b.beta[s] = a.beta[s].copy()
            if st.params.u1:
                b.qb[e + 1] = a.qb[e + 1].copy()
    return new_merged


def step(st: State, dt: float):
    """One full 2TDVP/p2TDVP timestep = half 1 + half 2 (AMB-14).

    Pairs evolved by the full dt at the end of half 1 are skipped in half 2
    (SURVEY.md O-9).
    """
    st.stats.w_step = 0.0
    st.stats.trunc_active = False
    merged = _half(st, dt, 1, set())
    _half(st, dt, 2, merged)
    st.stats.w_total += st.stats.w_step


# ----------------------------------------------------------------------------
# global state and measurement
# ----------------------------------------------------------------------------


def global_mps(st: State):
    """Owner copies: Psi_j from the segment owning site j; Lambda_b from the
    owner of site b (the left process owns a boundary bond, AMB-4)."""
    psi, lam = [None] * st.L, [None] * (st.L - 1)
    for seg in st.segs:
        for j in range(seg.s, seg.e + 1):
            psi[j] = seg.psi[j]
            if j < st.L - 1:
                lam[j] = seg.lam[j]
    return psi, lam


def chi_profile(st: State):
    _, lam = global_mps(st)
    return [1] + [len(l) for l in lam] + [1]


def _chain_tensors(psi, lam):
    """M_j = Psi_j V_j (j < L-1), M_{L-1} = Psi_{L-1}: |psi> = M_0 M_1 ... M_{L-1}."""
    L = len(psi)
    return [psi[j] * (1.0 / lam[j])[None, None, :] if j < L - 1 else psi[j] for j in range(L)]


def measure(st_or_mps, W=None):
    """Full-zipper <psi|psi>, <S^z_i> and E = <H> (normalised), any gauge (AMB-10).

    Accepts a State or (psi, lam) lists.  Uses transfer matrices, never a
    dense vector.
    """
    if isinstance(st_or_mps, State):
        psi, lam = global_mps(st_or_mps)
        W = st_or_mps.W
    else:
        psi, lam = st_or_mps
    M = _chain_tensors(psi, lam)
    L = len(M)
    # left transfer E_j = contraction of sites < j; right F_j of sites > j
    E = [None] * (L + 1)
    E[0] = np.ones((1, 1), dtype=np.complex128)
    for j in range(L):
        # E'[b,b'] = sum conj(M[a,s,b]) E[a,a'] M[a',s,b']
        E[j + 1] = np.tensordot(M[j].conj(), np.tensordot(E[j], M[j], axes=(1, 0)), axes=([0, 1], [0, 1]))
    F = [None] * (L + 1)
    F[L] = np.ones((1, 1), dtype=np.complex128)
    for j in range(L - 1, -1, -1):
        # F'[a,a'] = sum conj(M[a,s,b]) M[a',s,b'] F[b,b']
        F[j] = np.tensordot(M[j].conj(), np.tensordot(M[j], F[j + 1], axes=(2, 1)), axes=([1, 2], [1, 2]))
    nrm = float(np.real(E[L][0, 0]))
    sz = np.zeros(L)
    Sz = np.diag([0.5, -0.5]).astype(np.complex128)
    for j in range(L):
        X = np.tensordot(E[j], M[j], axes=(1, 0))            # [a, s, b']
        X = np.tensordot(X, Sz, axes=(1, 1))                  # [a, b', s]  (Sz[s,t] M[.,t,.])
        Y = np.tensordot(M[j].conj(), X, axes=([0, 1], [0, 2]))  # [b, b']
        sz[j] = float(np.real(np.sum(Y * F[j + 1]))) / nrm
    energy = None
    if W is not None:
        beta = np.ones((1, 1, 1), dtype=np.complex128)
        for j in range(L):
            beta = env_left(beta, M[j], W[j])
        energy = float(np.real(beta[0, 0, 0])) / nrm
    return dict(norm=nrm, sz=sz, energy=energy)


def to_dense(psi, lam):
    """Dense state vector (L <= ~16), site 0 most significant."""
    M = _chain_tensors(psi, lam)
    v = M[0].reshape(M[0].shape[1], M[0].shape[2])
    for j in range(1, len(M)):
        v = np.tensordot(v, M[j], axes=(v.ndim - 1, 0))
        v = v.reshape(-1, M[j].shape[2])
    return v.reshape(-1)


# ----------------------------------------------------------------------------
# literal serial sweep (PAPER.md:430 as written), independent of App. A code
# ----------------------------------------------------------------------------


def serial_step_literal(psi, lam, W, beta, gamma, dt, params: Params):
    """One serial 2TDVP step on global lists, exactly as PAPER.md:430 reads.

    "sites 1 and 2 are evolved forwards by half a timestep; site 2 is evolved
    backwards...; until the rightmost pair ... evolve the rightmost pair just
    once by a full timestep"; then the mirror sweep R->L.  Mutates the lists.
    Returns the step's discarded weight.
    """
    L = len(psi)
    tau_h, tau_f = -0.5j * dt, -1.0j * dt
    wsum = 0.0

    def pair(j, tau):
        nonlocal wsum
        th = merge_theta(psi[j], 1.0 / lam[j], psi[j + 1])
        th2 = expm_lanczos(lambda x: apply_h2(beta[j], W[j], W[j + 1], gamma[j + 1], x), th, tau,
                           params.krylov_k, params.krylov_tol)
        pl, S, pr, w, _, _ = svd_truncate(th2, params)
        psi[j], lam[j], psi[j + 1] = pl, S, pr
        wsum += w

    def back(j):
        psi[j] = expm_lanczos(lambda x: apply_h1(beta[j], W[j], gamma[j], x), psi[j], 0.5j * dt,
                              params.krylov_k, params.krylov_tol)

    # left-to-right sweep
    for j in range(L - 1):
        if j < L - 2:
            pair(j, tau_h)
            beta[j + 1] = env_left(beta[j], psi[j] * (1.0 / lam[j])[None, None, :], W[j])
            back(j + 1)
        else:
            pair(j, tau_f)  # rightmost pair once by the full timestep
            gamma[j] = env_right(gamma[j + 1], (1.0 / lam[j])[:, None, None] * psi[j + 1], W[j + 1])
    # right-to-left sweep (mirror image, first pair already done)
    for j in range(L - 2, -1, -1):
        if j < L - 2:
            pair(j, tau_h)
            gamma[j] = env_right(gamma[j + 1], (1.0 / lam[j])[:, None, None] * psi[j + 1], W[j + 1])
        if j > 0:
            back(j)
    return wsum
