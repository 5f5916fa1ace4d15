"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module is the ONLY code both sides use.  It builds *inputs*: product
states, random inverse-canonical MPS, and the Hamiltonian MPO tensors W_j.
It contains none of the method's arithmetic (no environments, no H_eff,
no Lanczos, no SVD truncation, no sweeps).

Conventions (SURVEY.md §8 "Conventions"):
  * spin-1/2, basis index 0 = up (S^z=+1/2), 1 = down; S = sigma/2.
  * Psi_j has shape (chi_l, d, chi_r), complex128, row-major.
  * Lambda_j (bond j between sites j and j+1) is float64, descending, > 0.
  * W_j has shape (D_l, d_out, d_in, D_r) with W[w, s, t, w'] = <s|O|t>.
  * MPO finite-state-machine layout: channel 0 = "done" (identity to the
    right), channel D-1 = "not started" (identity to the left); first site is
    row D-1 of the bulk W, last site is column 0 (§II.C).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

D_PHYS = 2

# single-site operators (input definitions of the model)
ID2 = np.eye(2, dtype=np.complex128)
SP = np.array([[0, 1], [0, 0]], dtype=np.complex128)  # S+ = |up><down|
SM = np.array([[0, 0], [1, 0]], dtype=np.complex128)  # S-
SZ = np.array([[0.5, 0], [0, -0.5]], dtype=np.complex128)
SX = 0.5 * (SP + SM)
SY = -0.5j * (SP - SM)


@dataclass
class MPS:
    """Inverse-canonical MPS input: Psi_0 V_0 Psi_1 ... V_{L-2} Psi_{L-1}.

    PAPER.md:357-365 (§II.B): V_j = Lambda_j^{-1}; every Psi_j is an
    orthogonality centre.
    """

    psi: list  # L arrays (chi_{j-1}, d, chi_j)
    lam: list  # L-1 float64 arrays (chi_j,)

    @property
    def L(self) -> int:
        return len(self.psi)

    def chi(self) -> list:
        """Bond dims including the trivial ends: length L+1."""
        return [1] + [p.shape[2] for p in self.psi[:-1]] + [1]

    def copy(self) -> "MPS":
        return MPS([p.copy() for p in self.psi], [l.copy() for l in self.lam])


# ----------------------------------------------------------------------------
# product states (chi = 1, trivially inverse canonical)
# ----------------------------------------------------------------------------

def product_mps(vectors) -> MPS:
    psi = []
    for v in vectors:
        v = np.asarray(v, dtype=np.complex128)
        v = v / np.linalg.norm(v)
        psi.append(v.reshape(1, D_PHYS, 1).copy())
    lam = [np.ones(1) for _ in range(len(psi) - 1)]
    return MPS(psi, lam)


def neel_mps(L: int) -> MPS:
    """Neel state: up on even sites (SURVEY.md §8 conventions)."""
    return product_mps([[1, 0] if i % 2 == 0 else [0, 1] for i in range(L)])


def all_up_mps(L: int) -> MPS:
    return product_mps([[1, 0]] * L)


def bloch_mps(L: int, seed: int = 0) -> MPS:
    """Seeded uniform-on-sphere product state.

    PCG64(seed); per site, in order: cos(theta) ~ U[-1, 1], phi ~ U[0, 2 pi).
    Site vector (cos(theta/2), e^{i phi} sin(theta/2)).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    vecs = []
    for _ in range(L):
        ct = rng.uniform(-1.0, 1.0)
        phi = rng.uniform(0.0, 2.0 * math.pi)
        th = math.acos(ct)
        vecs.append([math.cos(th / 2), complex(math.cos(phi), math.sin(phi)) * math.sin(th / 2)])
    return product_mps(vecs)


def single_flip_mps(L: int, sites) -> MPS:
    """All-up state with the listed sites flipped down (magnon-sector tests)."""
    sites = set(sites)
    return product_mps([[0, 1] if i in sites else [1, 0] for i in range(L)])


def saturated_chi_profile(L: int, chi: int) -> list:
    """chi_j = min(2^(j+1), 2^(L-j-1), chi) for bonds j = 0..L-2."""
    out = []
    for j in range(L - 1):
        a = 2 ** min(j + 1, 62)
        b = 2 ** min(L - j - 1, 62)
        out.append(int(min(a, b, chi)))
    return out


def random_canonical_mps(L: int, chi: int, seed: int = 2) -> MPS:
    """Random inverse-canonical MPS with a saturated bond profile.

    Seeded complex-normal tensors with chi_j = min(2^(j+1), 2^(L-j-1), chi),
    brought to inverse-canonical form by `canonicalize`.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    dims = [1] + saturated_chi_profile(L, chi) + [1]
    M = []
    for j in range(L):
        shp = (dims[j], D_PHYS, dims[j + 1])
        M.append(rng.standard_normal(shp) + 1j * rng.standard_normal(shp))
    return canonicalize(M)


def canonicalize(M) -> MPS:
    """Exact re-gauging of a chain M_0 ... M_{L-1} into inverse-canonical form.

    A QR sweep L->R, then an SVD sweep R->L giving Lambda_j and right-
    orthonormal B_j; Psi_0 = normalised first tensor, Psi_j = Lambda_{j-1} B_j
    (so Psi_0 V_0 Psi_1 ... = Psi_0 B_1 B_2 ...).  The state is normalised.
    Input preparation, not part of the TDVP method.
    """
    M = [np.asarray(m, dtype=np.complex128).copy() for m in M]
    L = len(M)
    for j in range(L - 1):
        cl, d, cr = M[j].shape
        q, r = np.linalg.qr(M[j].reshape(cl * d, cr))
        k = q.shape[1]
        M[j] = q.reshape(cl, d, k)
        # the overall scale is normalised away below; keep it O(1) so long
        # chains at large chi do not overflow
        M[j + 1] = np.tensordot(r / np.linalg.norm(r), M[j + 1], axes=(1, 0))
    lam = [None] * (L - 1)
    for j in range(L - 1, 0, -1):
        cl, d, cr = M[j].shape
        u, s, vh = np.linalg.svd(M[j].reshape(cl, d * cr), full_matrices=False)
        k = int(np.count_nonzero(s > s[0] * 1e-14))
        u, s, vh = u[:, :k], s[:k], vh[:k]
        M[j] = vh.reshape(k, d, cr)  # right-orthonormal B_j
        M[j - 1] = np.tensordot(M[j - 1], u * s[None, :], axes=(2, 0))
        lam[j - 1] = s
    nrm = np.linalg.norm(M[0])
    psi = [M[0] / nrm]
    lam = [l / nrm for l in lam]
    for j in range(1, L):
        psi.append(lam[j - 1][:, None, None] * M[j])
    return MPS(psi, lam)


def magnon_superposition_mps(L: int, seed: int = 3):
    """sum_i c_i |down at i> (random c_i) as a chi = 2 MPS, inverse-canonical.

    Returns (MPS, c).

    Finite-state tensors: channel 0 = "no magnon yet", 1 = "magnon placed".
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    c = rng.standard_normal(L) + 1j * rng.standard_normal(L)
    M = []
    for i in range(L):
        A = np.zeros((2, 2, 2), dtype=np.complex128)
        A[0, 0, 0] = 1.0
        A[0, 1, 1] = c[i]
        A[1, 0, 1] = 1.0
        if i == 0:
            A = A[0:1]
        if i == L - 1:
            A = A[:, :, 1:2]
        M.append(A)
    return canonicalize(M), c


# ----------------------------------------------------------------------------
# Hamiltonian MPOs (§II.C; SURVEY.md §8 "Exact MPO layout")
# ----------------------------------------------------------------------------

# channel types t: (P, Q, g) -> string P_i ... Q_k with weight g
_TERMS = ((SM, SP, 0.5), (SP, SM, 0.5), (SZ, SZ, None))  # g for Sz Sz is Delta


def mpo_xxz_expsum(L: int, a, lam, Delta: float, J: float = 1.0):
    """MPO of H = sum_{i<k} J(k-i) [1/2 (S+_i S-_k + S-_i S+_k) + Delta Sz_i Sz_k]
    with J(r) = J * sum_kappa a_kappa lam_kappa^(r-1)  (D = 3K + 2).

    Bulk W: W[0,0] = W[D-1,D-1] = I; W[D-1, c] = a g P; W[c, c] = lam I;
    W[c, 0] = Q, with c(t, kappa) = 1 + 3 kappa + t.
    """
    a = np.asarray(a, dtype=np.float64) * J
    lam = np.asarray(lam, dtype=np.float64)
    K = len(a)
    D = 3 * K + 2
    W = np.zeros((D, 2, 2, D), dtype=np.complex128)
    W[0, :, :, 0] = ID2
    W[D - 1, :, :, D - 1] = ID2
    for k in range(K):
        for t, (P, Q, g) in enumerate(_TERMS):
            gg = Delta if g is None else g
            c = 1 + 3 * k + t
            W[D - 1, :, :, c] = a[k] * gg * P
            W[c, :, :, c] = lam[k] * ID2
            W[c, :, :, 0] = Q
    return _open_chain(W, L)


def mpo_xxz_nn(L: int, Delta: float, J: float = 1.0):
    """Nearest-neighbour XXZ: the K=1, a=1, lam=0 case (D = 5, nnz(W) = 12)."""
    return mpo_xxz_expsum(L, [1.0], [0.0], Delta, J)


def mpo_onsite(L: int, op):
    """One-body H = sum_i op_i (D = 2), used by pin P11."""
    op = np.asarray(op, dtype=np.complex128)
    W = np.zeros((2, 2, 2, 2), dtype=np.complex128)
    W[0, :, :, 0] = ID2
    W[1, :, :, 1] = ID2
    W[1, :, :, 0] = op
    return _open_chain(W, L)


def mpo_zero(L: int):
    """H = 0 as a D=1 MPO with zero tensors (pin P12)."""
    return [np.zeros((1, 2, 2, 1), dtype=np.complex128) for _ in range(L)]


def _open_chain(W, L):
    D = W.shape[0]
    first = W[D - 1:D, :, :, :].copy()
    last = W[:, :, :, 0:1].copy()
    if L == 1:
        return [W[D - 1:D, :, :, 0:1].copy()]
    return [first] + [W.copy() for _ in range(L - 2)] + [last]


def fit_expsum(rmax: int = 100, K: int = 9, power: float = 2.0):
    """Deterministic matrix-pencil fit of 1/r^power on r = 1..rmax by
    sum_kappa a_kappa lam_kappa^(r-1)  (Pirvu).

    Returns (a, lam, max_abs_err, max_rel_err).  Input generation only.
    """
    r = np.arange(1, rmax + 1, dtype=np.float64)
    y = r ** (-power)
    N = rmax
    Lp = N // 2
    Y = np.array([y[i:i + Lp + 1] for i in range(N - Lp)])
    _, _, vh = np.linalg.svd(Y, full_matrices=False)
    Vk = vh[:K].conj().T
    V1, V2 = Vk[:-1], Vk[1:]
    z = np.linalg.eigvals(np.linalg.pinv(V1) @ V2)
    if np.max(np.abs(z.imag)) > 1e-8:
        raise RuntimeError("matrix-pencil fit produced complex poles")
    z = np.sort(z.real)[::-1]
    Vand = z[None, :] ** (r[:, None] - 1.0)
    a, *_ = np.linalg.lstsq(Vand, y, rcond=None)
    fit = Vand @ a
    err = np.abs(fit - y)
    return a, z, float(err.max()), float((err / y).max())


def expsum_J(a, lam, r):
    r = np.asarray(r, dtype=np.float64)
    return (np.asarray(a)[None, :] * np.asarray(lam)[None, :] ** (r[:, None] - 1.0)).sum(axis=1)


# ----------------------------------------------------------------------------
# benchmark configs (BASELINE.json "configs")
# ----------------------------------------------------------------------------

def config(name: str):
    """Return dict(L, mpo, mps, chi_max, eps, dt, steps, segments) for a config."""
    if name == "c1":
        L = 10
        return dict(L=L, mpo=mpo_xxz_nn(L, 1.0), mps=neel_mps(L), chi_max=32, eps=1e-12,
                    dt=0.05, steps=20, segments=[1], Delta=1.0)
    if name == "c2":
        L = 64
        return dict(L=L, mpo=mpo_xxz_nn(L, 0.5), mps=neel_mps(L), chi_max=128, eps=1e-10,
                    dt=0.05, steps=40, segments=[1], Delta=0.5)
    if name == "c3":
        L = 128
        return dict(L=L, mpo=mpo_xxz_nn(L, 1.5), mps=neel_mps(L), chi_max=512, eps=1e-10,
                    dt=0.02, steps=20, segments=[8], Delta=1.5)
    if name == "c4":
        L = 100
        a, lam, _, _ = fit_expsum(100, 9, 2.0)
        return dict(L=L, mpo=mpo_xxz_expsum(L, a, lam, 1.0), mps=bloch_mps(L, 0), chi_max=256,
                    eps=1e-12, dt=0.02, steps=10, segments=[1, 2, 4], Delta=1.0)
    if name == "c5":
        L = 256
        return dict(L=L, mpo=mpo_xxz_nn(L, 1.0), mps=neel_mps(L), chi_max=1024, eps=1e-12,
                    dt=0.05, steps=10, segments=[1, 2, 4, 8], Delta=1.0)
    raise KeyError(name)


def random_complex(shape, rng):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


# ----------------------------------------------------------------------------
# U(1) (S^z_tot-conserving) synthetic inputs: a random MPS
# of definite total S^z whose bond indices carry charges q = 2 S^z of the
# sites to their left, Psi_j[a, s, b] = 0 unless q_b = q_a + c(s) with
# c(up) = +1, c(down) = -1.  Input preparation only.
# ----------------------------------------------------------------------------

U1_CS = (1, -1)


def _u1_bond_charges(L: int, chi: int, total: int = 0):
    """Charge multiplicities of a saturated charge-definite bond profile: bond
    position k (left of site k) gets the charges q of k spins that the L - k
    spins to its right can complete to `total`, each with multiplicity at
    most min(#left states, #right states) of that charge, the bond dimension
    min(2^k, 2^(L-k), chi) spread over the charges in proportion to those
    counts (largest first)."""
    out = []
    for k in range(L + 1):
        cap = {}
        for nup in range(k + 1):
            q = 2 * nup - k
            rq = total - q  # charge the right part must carry
            if (L - k + rq) % 2 or abs(rq) > L - k:
                continue
            cap[q] = min(math.comb(k, nup), math.comb(L - k, (L - k + rq) // 2))
        target = min(2 ** min(k, 62), 2 ** min(L - k, 62), chi, sum(cap.values()))
        tot = sum(cap.values())
        mult = {q: min(c, int(target * c / tot)) for q, c in cap.items()}
        left = target - sum(mult.values())
        for q in sorted(cap, key=lambda x: (-cap[x], x)):
            if left <= 0:
                break
            add = min(left, cap[q] - mult[q])
            mult[q] += add
            left -= add
        out.append(np.array(sorted(q for q, m in mult.items() for _ in range(m)), dtype=np.int64))
    return out


def random_u1_mps(L: int, chi: int, seed: int = 2, total: int = 0) -> MPS:
    """Random inverse-canonical MPS of definite total charge (2 S^z_tot = total)
    with a saturated charge-resolved bond profile; seeded complex-normal
    entries on the allowed blocks, re-gauged by canonicalize_u1."""
    rng = np.random.Generator(np.random.PCG64(seed))
    q = _u1_bond_charges(L, chi, total)
    M = []
    for j in range(L):
        t = np.zeros((len(q[j]), D_PHYS, len(q[j + 1])), dtype=np.complex128)
        for s in range(D_PHYS):
            mask = (q[j][:, None] + U1_CS[s]) == q[j + 1][None, :]
            t[:, s, :] = np.where(mask, random_complex(mask.shape, rng), 0.0)
        M.append(t)
    return canonicalize_u1(M, q)


def canonicalize_u1(M, q) -> MPS:
    """canonicalize() done sector by sector, so that every tensor keeps exact
    zeros outside its charge blocks (the block structure is what the U(1)
    path of both oracle and library infer the charges from).  Bond indices
    are ordered by descending Schmidt value."""
    M = [np.asarray(m, dtype=np.complex128).copy() for m in M]
    q = [np.asarray(x, dtype=np.int64).copy() for x in q]
    L = len(M)
    # QR sweep L -> R, per sector of the right bond
    for j in range(L - 1):
        cl, d, cr = M[j].shape
        A = M[j].reshape(cl * d, cr)
        rq = (q[j][:, None] + np.array(U1_CS[:d])[None, :]).reshape(-1)
        Qs, Rs, newq = [], [], []
        for Q in sorted(set(q[j + 1].tolist())):
            rows, cols = np.nonzero(rq == Q)[0], np.nonzero(q[j + 1] == Q)[0]
            qq, rr = np.linalg.qr(A[np.ix_(rows, cols)])
            Qs.append((rows, qq))
            Rs.append((cols, rr))
            newq += [Q] * qq.shape[1]
        k = len(newq)
        An = np.zeros((cl * d, k), dtype=np.complex128)
        R = np.zeros((k, cr), dtype=np.complex128)
        off = 0
        for (rows, qq), (cols, rr) in zip(Qs, Rs):
            An[rows, off:off + qq.shape[1]] = qq
            R[off:off + rr.shape[0], cols] = rr
            off += qq.shape[1]
        M[j] = An.reshape(cl, d, k)
        M[j + 1] = np.tensordot(R / np.linalg.norm(R), M[j + 1], axes=(1, 0))
        q[j + 1] = np.array(newq, dtype=np.int64)
    # SVD sweep R -> L, per sector of the left bond
    lam = [None] * (L - 1)
    for j in range(L - 1, 0, -1):
        cl, d, cr = M[j].shape
        A = M[j].reshape(cl, d * cr)
        cq = (q[j + 1][None, :] - np.array(U1_CS[:d])[:, None]).reshape(-1)
        trip = []
        for Q in sorted(set(q[j].tolist())):
            rows, cols = np.nonzero(q[j] == Q)[0], np.nonzero(cq == Q)[0]
            u, s, vh = np.linalg.svd(A[np.ix_(rows, cols)], full_matrices=False)
            for kk in range(len(s)):
                trip.append((s[kk], Q, rows, u[:, kk], cols, vh[kk]))
        trip.sort(key=lambda t: (-t[0], t[1]))
        smax = trip[0][0]
        trip = [t for t in trip if t[0] > 1e-14 * smax]
        k = len(trip)
        U = np.zeros((cl, k), dtype=np.complex128)
        B = np.zeros((k, d * cr), dtype=np.complex128)
        s_ = np.zeros(k)
        for kk, (s, Q, rows, u, cols, vh) in enumerate(trip):
            U[rows, kk] = u
            B[kk, cols] = vh
            s_[kk] = s
        M[j] = B.reshape(k, d, cr)
        M[j - 1] = np.tensordot(M[j - 1], U * s_[None, :], axes=(2, 0))
        lam[j - 1] = s_
        q[j] = np.array([t[1] for t in trip], dtype=np.int64)
    nrm = np.linalg.norm(M[0])
    psi = [M[0] / nrm]
    lam = [l / nrm for l in lam]
    for j in range(1, L):
        psi.append(lam[j - 1][:, None, None] * M[j])
    return MPS(psi, lam)
