"""Exact references that pin the oracle (TEST INFRASTRUCTURE ONLY).

Written from the model definition, independent of the MPO construction:
  H = sum_{i<k} J(k-i) [1/2 (S+_i S-_k + S-_i S+_k) + Delta Sz_i Sz_k]
(at Delta = 1, J = 1/r^2 this is PAPER.md:645 Eq. HaldaneHamiltonian).
Site 0 is the most significant bit of the dense index; bit value 0 = up.
"""
from __future__ import annotations

from itertools import combinations

import numpy as np
import scipy.sparse as sp


def _site_op(op, i, L):
    """op acting on site i of L as a sparse 2^L matrix (Kronecker product)."""
    out = sp.identity(1, dtype=np.complex128, format="csr")
    I2 = sp.identity(2, dtype=np.complex128, format="csr")
    for k in range(L):
        out = sp.kron(out, sp.csr_matrix(op) if k == i else I2, format="csr")
    return out


_SP = np.array([[0, 1], [0, 0]], dtype=np.complex128)
_SM = _SP.T.copy()
_SZ = np.diag([0.5, -0.5]).astype(np.complex128)


def dense_hamiltonian(L, Jr, Delta):
    """Dense H for couplings Jr(r) (callable, r >= 1; 0 beyond range)."""
    sps = [_site_op(_SP, i, L) for i in range(L)]
    sms = [_site_op(_SM, i, L) for i in range(L)]
    szs = [_site_op(_SZ, i, L) for i in range(L)]
    H = sp.csr_matrix((2 ** L, 2 ** L), dtype=np.complex128)
    for i in range(L):
        for k in range(i + 1, L):
            J = Jr(k - i)
            if J == 0.0:
                continue
            H = H + J * (0.5 * (sps[i] @ sms[k] + sms[i] @ sps[k]) + Delta * (szs[i] @ szs[k]))
    return H.toarray()


def dense_onsite(L, op):
    H = sp.csr_matrix((2 ** L, 2 ** L), dtype=np.complex128)
    for i in range(L):
        H = H + _site_op(np.asarray(op, dtype=np.complex128), i, L)
    return H.toarray()


def evolve(H, psi, t):
    """exp(-i H t) psi by Hermitian eigendecomposition."""
    e, U = np.linalg.eigh(H)
    return U @ (np.exp(-1j * e * t) * (U.conj().T @ psi))


def sz_dense(psi, L):
    """<S^z_i> of a dense vector (normalised)."""
    p = np.abs(psi.reshape([2] * L)) ** 2
    p = p / p.sum()
    out = np.zeros(L)
    for i in range(L):
        m = np.moveaxis(p, i, 0).reshape(2, -1).sum(axis=1)
        out[i] = 0.5 * (m[0] - m[1])
    return out


def product_dense(vecs):
    v = np.ones(1, dtype=np.complex128)
    for x in vecs:
        v = np.kron(v, np.asarray(x, dtype=np.complex128))
    return v / np.linalg.norm(v)


# ----------------------------------------------------------------------------
# free fermions (Delta = 0, nearest neighbour): pin P10
# ----------------------------------------------------------------------------


def free_fermion_sz(L, t, up_sites, J=1.0):
    """<S^z_i(t)> for H = J/2 sum (S+_i S-_{i+1} + h.c.) from a product state.

    Jordan-Wigner: S^z = n - 1/2 with n = 1 for up; the single-particle
    hopping matrix h_{i,i+1} = J/2; n_i(t) = sum_k |[e^{-iht}]_{ik}|^2 n_k(0)
    for an occupation-basis product state (no coherences).
    """
    h = np.zeros((L, L))
    for i in range(L - 1):
        h[i, i + 1] = h[i + 1, i] = 0.5 * J
    e, U = np.linalg.eigh(h)
    G = U @ np.diag(np.exp(-1j * e * t)) @ U.T
    n0 = np.zeros(L)
    n0[list(up_sites)] = 1.0
    return (np.abs(G) ** 2) @ n0 - 0.5


# ----------------------------------------------------------------------------
# magnon sectors (fixed number of down spins in an up background): pin P14
# ----------------------------------------------------------------------------


def magnon_hamiltonian(L, n_down, Jr, Delta):
    """H restricted to the sector with n_down flipped spins (basis = site sets)."""
    basis = [frozenset(c) for c in combinations(range(L), n_down)]
    index = {b: i for i, b in enumerate(basis)}
    n = len(basis)
    H = np.zeros((n, n), dtype=np.complex128)
    for idx, b in enumerate(basis):
        diag = 0.0
        for i in range(L):
            for k in range(i + 1, L):
                J = Jr(k - i)
                if J == 0.0:
                    continue
                zi = -0.5 if i in b else 0.5
                zk = -0.5 if k in b else 0.5
                diag += J * Delta * zi * zk
                # 1/2 (S+_i S-_k + S-_i S+_k): swaps an up/down pair
                if (i in b) != (k in b):
                    nb = (b - {i}) | {k} if i in b else (b - {k}) | {i}
                    H[index[nb], idx] += 0.5 * J
        H[idx, idx] += diag
    return H, basis


def magnon_sz(L, n_down, Jr, Delta, init_down, t):
    H, basis = magnon_hamiltonian(L, n_down, Jr, Delta)
    v = np.zeros(len(basis), dtype=np.complex128)
    v[basis.index(frozenset(init_down))] = 1.0
    v = evolve(H, v, t)
    prob = np.abs(v) ** 2
    sz = np.full(L, 0.5)
    for pb, b in zip(prob, basis):
        for i in b:
            sz[i] -= pb
    return sz
