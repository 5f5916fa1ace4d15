"""Smallest cases of every kernel family, for compute-sanitizer (one tool per run):
SVD (register Jacobi + cluster QR, and the DMMA block Jacobi forced small via
TDVP_SVD_BJ_MIN=32 set by the caller), Lanczos, H_eff, a 2-segment lane step,
a multi-device (repeated id) step, DMRG.  Exits 0 when every result is finite."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_06127_b200 as B  # noqa: E402
import tdvp_inputs as ti  # noqa: E402

rng = np.random.default_rng(0)
M = rng.standard_normal((72, 40)) + 1j * rng.standard_normal((72, 40))
pl, S, pr, w = B.svd_split(M, 20, eps=1e-10)
assert np.all(np.isfinite(S))
H = rng.standard_normal((24, 24))
H = H + H.T
v = rng.standard_normal(24) + 0j
assert np.all(np.isfinite(B.expm_lanczos_dense(H.astype(complex), v, -0.05j, K=8)))
L = 8
W = ti.mpo_xxz_nn(L, 0.5)
for devices, p in ((None, 2), ([0, 0], 2)):
    t = B.Tdvp(L, 2, 5, 8, devices=devices)
    t.set_params(eps=1e-10)
    t.set_mpo(W)
    mps = ti.random_canonical_mps(L, 8, seed=1)
    t.set_mps(mps.psi, mps.lam)
    t.step(0.05, p)
    assert np.all(np.isfinite(t.measure_sz()))
    t.close()
t = B.Tdvp(L, 2, 5, 8)
t.set_mpo(W)
t.set_mps(ti.neel_mps(L).psi, ti.neel_mps(L).lam)
assert np.all(np.isfinite(t.dmrg(1, 2)))
t.close()
print("sanitize case ok")
