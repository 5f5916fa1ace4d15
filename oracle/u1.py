"""U(1)-symmetric (S^z-conserving) block-sparse truncated SVD for the oracle
 -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's chi = 1024 runs use "symmetric block-sparse tensors"
(PAPER.md:643-651; :100 blocking tolerance).  For an S^z_tot-conserving MPO
and a state of definite S^z_tot every bond index b carries a charge q(b) =
2 S^z of the sites to its left, and Psi_j[a, s, b] != 0 only if
q(b) = q(a) + c(s), with c(up) = +1, c(down) = -1 (basis index 0 = up,
SURVEY.md §8 conventions).  The two-site matrix Theta[(a, s1), (s2, b)]
(AMB-17) is then block diagonal in the charge Q of the middle bond:
rows carry Q = q(a) + c(s1), columns Q = q(b) - c(s2).  Its SVD is the union
of the per-sector SVDs; the truncation rule O-7 (incl. AMB-9 / R-9b) acts on
the union of all sectors' singular values in descending order, exactly as on
the dense spectrum, and every kept singular vector lives in one sector, so
the new bond keeps definite charges.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg

from .tdvp import Params, truncation_rank

C_S = np.array([1, -1])  # 2 S^z of the local basis states (d = 2: up, down)


def infer_charges(psi):
    """Bond charges q[k] (k = 0..L, bond left of site k; q[0] = [0]) of an MPS
    whose tensors respect U(1), from their nonzero pattern.  Raises
    ValueError if a bond index is reachable with two different charges (the
    state is not of definite charge in this basis) or never (a zero column)."""
    L = len(psi)
    q = [np.zeros(1, dtype=np.int64)]
    for j in range(L):
        t = np.asarray(psi[j])
        cl, d, cr = t.shape
        qb = np.full(cr, np.iinfo(np.int64).min, dtype=np.int64)
        for a in range(cl):
            for s in range(d):
                for b in np.nonzero(t[a, s, :] != 0)[0]:
                    val = q[j][a] + C_S[s]
                    if qb[b] == np.iinfo(np.int64).min:
                        qb[b] = val
                    elif qb[b] != val:
                        raise ValueError(f"bond {j + 1} index {b}: charges {qb[b]} and {val}")
        if np.any(qb == np.iinfo(np.int64).min):
            raise ValueError(f"bond {j + 1}: an index with no nonzero entry")
        q.append(qb)
    return q


def svd_truncate_u1(theta, qa, qb, p: Params):
    """Sector-wise SVD split of theta (cl, d, d, cr) with left/right bond
    charges qa (cl), qb (cr): returns (psi_l, S, psi_r, w, r, chi_eps, q_mid)
    with the meaning of oracle.tdvp.svd_truncate plus q_mid, the charges of
    the kept singular vectors (the new middle bond)."""
    cl, d1, d2, cr = theta.shape
    M = theta.reshape(cl * d1, d2 * cr)
    if not np.all(np.isfinite(M)):
        raise FloatingPointError("non-finite Theta before SVD")
    rq = (np.asarray(qa)[:, None] + C_S[None, :d1]).reshape(-1)          # row (a, s1)
    cq = (np.asarray(qb)[None, :] - C_S[:d2, None]).reshape(-1)          # col (s2, b)
    trip = []  # (sigma, charge, k-in-sector, rows, cols, u, vh)
    for Q in sorted(set(rq.tolist()) & set(cq.tolist())):
        rows, cols = np.nonzero(rq == Q)[0], np.nonzero(cq == Q)[0]
        u, s, vh = scipy.linalg.svd(M[np.ix_(rows, cols)], full_matrices=False, lapack_driver="gesvd")
        for k in range(len(s)):
            trip.append((s[k], Q, k, rows, cols, u[:, k], vh[k]))
    # the dense spectrum in descending order (ties: sector charge, then index)
    trip.sort(key=lambda t: (-t[0], t[1], t[2]))
    sig = np.array([t[0] for t in trip])
    if len(sig) == 0 or sig[0] <= 0:
        raise FloatingPointError("all singular values zero")
    chi = truncation_rank(sig, p)
    w = float(np.sum(sig[chi:] ** 2))
    psi_l = np.zeros((cl * d1, chi), dtype=np.complex128)
    psi_r = np.zeros((chi, d2 * cr), dtype=np.complex128)
    for k in range(chi):
        s, Q, _, rows, cols, u, vh = trip[k]
        psi_l[rows, k] = u * s
        psi_r[k, cols] = s * vh
    eps = p.eps if p.eps > 0 else 1e-14
    chi_eps = int(np.count_nonzero(sig >= eps * sig[0]))
    q_mid = np.array([trip[k][1] for k in range(chi)], dtype=np.int64)
    return (psi_l.reshape(cl, d1, chi), sig[:chi].copy(), psi_r.reshape(chi, d2, cr), w, len(sig), chi_eps, q_mid)
