"""GPU parity: libtdvp (CUDA, through the C-ABI) against the CPU oracle.

Kernel level: every contraction of the hot path on random operands at ragged
sizes (several 64x64 tiles plus a tail), <= 1e-12 relative Frobenius.
Integrator level: <S^z_i>, E, norm and the chi profile after every step of
the same seeded runs with the same segment partition; 1e-9 absolute when no
truncation is active, 1e-6 otherwise (BASELINE.json north_star).
"""
import numpy as np
import pytest

import tdvp_inputs as ti
from oracle import tdvp as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1912_06127_b200 as pkg
    return pkg


def rc(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ------------------------------------------------------------------ kernels
@pytest.mark.parametrize("opA", "NTCR")
@pytest.mark.parametrize("opB", "NTCR")
def test_zgemm_all_ops(B, opA, opB):
    rng = np.random.default_rng(0)
    M, N, K = 131, 77, 203
    A = rc(rng, K, M) if opA in "TC" else rc(rng, M, K)
    Bm = rc(rng, N, K) if opB in "TC" else rc(rng, K, N)
    f = {"N": lambda x: x, "T": lambda x: x.T, "C": lambda x: x.conj().T, "R": lambda x: x.conj()}
    ref = f[opA](A) @ f[opB](Bm)
    out = B.zgemm(opA, opB, A, Bm)
    assert rel(out, ref) < 1e-14


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (8, 8, 4), (64, 64, 8), (65, 129, 257), (5, 3, 4096), (2048, 16, 640),
                                   (1024, 1280, 96), (1100, 1090, 300)])
def test_zgemm_shapes(B, M, N, K):
    rng = np.random.default_rng(M + N + K)
    A, Bm = rc(rng, M, K), rc(rng, K, N)
    assert rel(B.zgemm("N", "N", A, Bm), A @ Bm) < 1e-14


def _mpo_site(kind, rng):
    if kind == "nn":
        W = ti.mpo_xxz_nn(4, 0.7)[1]
    elif kind == "lr":
        a, lam, _, _ = ti.fit_expsum(100, 9, 2.0)
        W = ti.mpo_xxz_expsum(4, a, lam, 1.0)[1]
    else:
        W = rc(rng, 3, 2, 2, 4)
    return W


@pytest.mark.parametrize("cl,cr,kind", [(1, 2, "nn"), (37, 53, "nn"), (70, 66, "nn"), (33, 17, "lr"), (24, 24, "rand")])
def test_heff2_matches_oracle(B, cl, cr, kind):
    rng = np.random.default_rng(cl * 100 + cr)
    W1 = _mpo_site(kind, rng)
    W2 = _mpo_site(kind, rng) if kind != "rand" else rc(rng, 4, 2, 2, 3)
    Lenv = rc(rng, cl, W1.shape[0], cl)
    Renv = rc(rng, cr, W2.shape[3], cr)
    th = rc(rng, cl, 2, 2, cr)
    ref = O.apply_h2(Lenv, W1, W2, Renv, th)
    assert rel(B.apply_heff2(Lenv, W1, W2, Renv, th), ref) < 1e-13


@pytest.mark.parametrize("cl,cr,kind", [(1, 2, "nn"), (45, 70, "nn"), (19, 33, "lr"), (16, 9, "rand")])
def test_heff1_and_envs_match_oracle(B, cl, cr, kind):
    rng = np.random.default_rng(cl * 7 + cr)
    W = _mpo_site(kind, rng)
    Dl, Dr = W.shape[0], W.shape[3]
    Lenv, Renv = rc(rng, cl, Dl, cl), rc(rng, cr, Dr, cr)
    psi = rc(rng, cl, 2, cr)
    assert rel(B.apply_heff1(Lenv, W, Renv, psi), O.apply_h1(Lenv, W, Renv, psi)) < 1e-13
    assert rel(B.env_left(Lenv, psi, W), O.env_left(Lenv, psi, W)) < 1e-13
    assert rel(B.env_right(Renv, psi, W), O.env_right(Renv, psi, W)) < 1e-13


@pytest.mark.parametrize("n,K", [(32, 8), (300, 8), (7, 8), (64, 12)])
def test_lanczos_matches_oracle(B, n, K):
    rng = np.random.default_rng(n)
    A = rc(rng, n, n)
    H = (A + A.conj().T) / 2
    v = rc(rng, n)
    for tau in (-0.05j, 0.025j, -0.1j):
        ref = O.expm_lanczos(lambda x: H @ x, v, tau, K=K)
        out = B.expm_lanczos_dense(H, v, tau, K=K)
        assert rel(out, ref) < 1e-12


@pytest.mark.parametrize("m,n,chi_max", [(2, 2, 2), (8, 6, 6), (40, 72, 20), (128, 128, 64), (256, 200, 128),
                                         (66, 34, 40)])
def test_svd_split_matches_oracle(B, m, n, chi_max):
    rng = np.random.default_rng(m * n)
    M = rc(rng, m, n) * np.exp(-np.linspace(0, 30, n))[None, :]  # graded spectrum down to ~1e-13
    p = O.Params(chi_max=chi_max, eps=1e-10)
    pl_o, S_o, pr_o, w_o, _, _ = O.svd_truncate(M.reshape(m, 1, 1, n), p)
    pl, S, pr, w = B.svd_split(M, chi_max, eps=1e-10)
    assert len(S) == len(S_o)
    assert np.allclose(S, S_o, rtol=1e-11, atol=1e-14 * S_o[0])
    assert abs(w - w_o) <= 1e-12 * np.linalg.norm(M) ** 2
    # gauge-invariant: the truncated matrix Psi_L V Psi_R
    rec = (pl / S[None, :]) @ pr
    rec_o = pl_o.reshape(m, -1) @ np.diag(1 / S_o) @ pr_o.reshape(-1, n)
    assert rel(rec, rec_o) < 1e-10
    U = pl / S[None, :]
    assert np.abs(U.conj().T @ U - np.eye(len(S))).max() < 1e-12


@pytest.mark.parametrize("m,n,chi_max", [(600, 520, 300), (1024, 1024, 512), (512, 384, 384)])
def test_svd_split_grid_qr_sizes(B, m, n, chi_max):
    """256 < n <= 1024: the cooperative-grid look-ahead QR preconditioner and
    the register-resident Jacobi variants for X <= 512 / 1024 rows."""
    rng = np.random.default_rng(m + n)
    M = rc(rng, m, n) * np.exp(-np.linspace(0, 25, n))[None, :]
    S_ref = np.linalg.svd(M, compute_uv=False)
    pl, S, pr, w = B.svd_split(M, chi_max, eps=1e-10)
    k = len(S)
    assert k == min(chi_max, int(np.count_nonzero(S_ref >= 1e-10 * S_ref[0])))
    assert np.allclose(S, S_ref[:k], rtol=1e-10, atol=1e-13 * S_ref[0])
    assert abs(w - np.sum(S_ref[k:] ** 2)) <= 1e-10 * np.sum(S_ref ** 2)
    U = pl / S[None, :]
    assert np.abs(U.conj().T @ U - np.eye(k)).max() < 1e-11
    Wt = pr / S[:, None]
    assert np.abs(Wt @ Wt.conj().T - np.eye(k)).max() < 1e-11


def test_svd_split_large_blocked_qr(B):
    """mr in (1024, 2048]: blocked Householder QR preconditioner (panel width 4)
    and the streaming Jacobi; graded spectrum down to 1e-12."""
    rng = np.random.default_rng(17)
    m, n, chi_max = 1500, 1100, 600
    M = rc(rng, m, n) * np.exp(-np.linspace(0, 27, n))[None, :]
    p = O.Params(chi_max=chi_max, eps=1e-10)
    pl_o, S_o, pr_o, w_o, _, _ = O.svd_truncate(M.reshape(m, 1, 1, n), p)
    pl, S, pr, w = B.svd_split(M, chi_max, eps=1e-10)
    assert len(S) == len(S_o)
    assert np.allclose(S, S_o, rtol=1e-10, atol=1e-14 * S_o[0])
    U = pl / S[None, :]
    assert np.abs(U.conj().T @ U - np.eye(len(S))).max() < 1e-11
    rec = (pl / S[None, :]) @ pr
    rec_o = pl_o.reshape(m, -1) @ np.diag(1 / S_o) @ pr_o.reshape(-1, n)
    assert rel(rec, rec_o) < 1e-9


def test_svd_split_chi1024_shape(B):
    """The chi = 1024 two-site shape (2048 x 2048, configs[4]): blocked QR
    preconditioner + streaming Jacobi (BW = 8, register-tiled Gram/apply),
    truncated to chi_max = 1024 with eps = 1e-12 (sampled checks: sigma,
    discarded weight, orthonormality of the kept left factor)."""
    rng = np.random.default_rng(23)
    n, chi_max = 2048, 1024
    M = rc(rng, n, n) * np.exp(-np.linspace(0, 20, n))[None, :]
    S_ref = np.linalg.svd(M, compute_uv=False)
    pl, S, pr, w = B.svd_split(M, chi_max, eps=1e-12)
    k = len(S)
    assert k == min(chi_max, int(np.count_nonzero(S_ref >= 1e-12 * S_ref[0])))
    assert np.allclose(S, S_ref[:k], rtol=1e-10, atol=1e-13 * S_ref[0])
    assert abs(w - np.sum(S_ref[k:] ** 2)) <= 1e-10 * np.sum(S_ref ** 2)
    U = pl[:, :64] / S[None, :64]
    assert np.abs(U.conj().T @ U - np.eye(64)).max() < 1e-11


def test_svd_degenerate_and_rank_deficient(B):
    rng = np.random.default_rng(5)
    Q1, _ = np.linalg.qr(rc(rng, 20, 20))
    Q2, _ = np.linalg.qr(rc(rng, 12, 12))
    s = np.array([3.0, 2.0, 2.0, 2.0, 1.0, 0.5] + [0.0] * 6)
    M = Q1[:, :12] @ np.diag(s) @ Q2.conj().T
    for chi_max in (3, 4, 12):
        p = O.Params(chi_max=chi_max, eps=1e-12)
        _, S_o, _, w_o, _, _ = O.svd_truncate(M.reshape(20, 1, 1, 12), p)
        _, S, _, w = B.svd_split(M, chi_max, eps=1e-12)
        assert len(S) == len(S_o) and np.allclose(S, S_o, rtol=1e-12)
        assert abs(w - w_o) < 1e-12


# --------------------------------------------------------------- integrator
def gpu_run(B, mps, W, chi_max, eps, dt, steps, p, krylov_k=8, every=1):
    D = max(w.shape[3] for w in W)
    t = B.Tdvp(len(W), 2, max(D, max(w.shape[0] for w in W)), chi_max)
    t.set_params(eps=eps, krylov_k=krylov_k)
    t.set_mpo(W)
    t.set_mps(mps.psi, mps.lam)
    out = []
    for n in range(steps):
        t.step(dt, p)
        if (n + 1) % every == 0 or n + 1 == steps:
            out.append(dict(sz=t.measure_sz(), E=t.measure_energy(), norm=t.measure_norm(), chi=t.chi(),
                            stats=t.stats()))
    t.close()
    return out


def oracle_run(mps, W, chi_max, eps, dt, steps, p, krylov_k=8, every=1):
    st = O.init_state(mps, W, O.Params(chi_max=chi_max, eps=eps, krylov_k=krylov_k), p)
    out = []
    for n in range(steps):
        O.step(st, dt)
        if (n + 1) % every == 0 or n + 1 == steps:
            m = O.measure(st)
            out.append(dict(sz=m["sz"], E=m["energy"], norm=m["norm"], chi=O.chi_profile(st),
                            trunc=st.stats.trunc_active, w=st.stats.w_step))
    return out


def compare(g, o, tol_untrunc=1e-9, tol_trunc=1e-6):
    trunc = False
    for a, b in zip(g, o):
        trunc = trunc or b["trunc"]
        tol = tol_trunc if trunc else tol_untrunc
        assert a["chi"] == b["chi"], (a["chi"], b["chi"])
        assert np.abs(a["sz"] - b["sz"]).max() < tol
        assert abs(a["E"] - b["E"]) < tol
        assert abs(a["norm"] - b["norm"]) < tol


def test_config1_serial_untruncated(B):
    cfg = ti.config("c1")
    args = (cfg["mps"], cfg["mpo"], cfg["chi_max"], cfg["eps"], cfg["dt"], cfg["steps"], 1)
    g, o = gpu_run(B, *args), oracle_run(*args)
    compare(g, o)
    assert not any(x["trunc"] for x in o)


@pytest.mark.parametrize("p", [2, 4])
def test_segmented_small(B, p):
    L = 16
    mps, W = ti.neel_mps(L), ti.mpo_xxz_nn(L, 0.5)
    args = (mps, W, 32, 1e-12, 0.05, 10, p)
    compare(gpu_run(B, *args), oracle_run(*args))


def test_long_range_random_state(B):
    L = 20
    a, lam, _, _ = ti.fit_expsum(100, 9, 2.0)
    args = (ti.bloch_mps(L, 0), ti.mpo_xxz_expsum(L, a, lam, 1.0), 16, 1e-12, 0.02, 4, 2)
    compare(gpu_run(B, *args), oracle_run(*args))


def test_truncated_saturated(B):
    L = 12
    mps = ti.random_canonical_mps(L, 8, seed=2)
    args = (mps, ti.mpo_xxz_nn(L, 0.5), 8, 1e-10, 0.05, 3, 1)
    g, o = gpu_run(B, *args), oracle_run(*args)
    assert o[0]["trunc"]
    compare(g, o)


def test_one_body_exact_on_gpu(B):
    L, h = 8, 0.7
    g = gpu_run(B, ti.neel_mps(L), ti.mpo_onsite(L, h * ti.SX), 8, 1e-12, 0.1, 10, 2)
    exact = np.array([0.5 if i % 2 == 0 else -0.5 for i in range(L)]) * np.cos(h * 1.0)
    assert np.abs(g[-1]["sz"] - exact).max() < 1e-12


@pytest.mark.parametrize("lanes", ["1", "0"])
def test_explicit_partition_matches_oracle(B, lanes, monkeypatch):
    """N4: an explicit (uneven, load-balanced) partition on the GPU equals the
    oracle run on the same partition; both executors (lanes / round-robin)."""
    monkeypatch.setenv("TDVP_LANES", lanes)
    L = 16
    mps, W = ti.random_canonical_mps(L, 8, seed=4), ti.mpo_xxz_nn(L, 0.5)
    chi = [1] + [len(x) for x in mps.lam] + [1]
    bounds = B.balanced_partition(L, 4, chi)
    assert bounds != B.partition(L, 4)
    t = B.Tdvp(L, 2, 5, 8)
    t.set_params(eps=1e-10)
    t.set_mpo(W)
    t.set_mps(mps.psi, mps.lam)
    t.set_partition(bounds)
    st = O.init_state(mps, W, O.Params(chi_max=8, eps=1e-10), 4, bounds)
    for _ in range(3):
        t.step(0.05, 4)
        O.step(st, 0.05)
        m = O.measure(st)
        assert t.chi() == O.chi_profile(st)
        assert np.abs(t.measure_sz() - m["sz"]).max() < 1e-6
        assert abs(t.measure_energy() - m["energy"]) < 1e-6
    t.set_partition(None)  # back to the uniform rule: state kept, re-laid out
    t.step(0.05, 4)
    psi, lam = O.global_mps(st)
    st2 = O.init_state(ti.MPS(psi, lam), W, O.Params(chi_max=8, eps=1e-10), 4)
    O.step(st2, 0.05)
    assert np.abs(t.measure_sz() - O.measure(st2)["sz"]).max() < 1e-6
    t.close()


@pytest.mark.parametrize("p", [1, 2])
def test_paper_mode_krylov_tol_matches_oracle(B, p):
    """krylov_tol > 0 (paper mode: max 8 vectors, tolerance
    1e-6): the device-side stopping rule equals the oracle's, so the runs agree
    like the fixed-K runs; and they differ from fixed K = 8 by at most ~tol."""
    L = 12
    mps, W = ti.random_canonical_mps(L, 8, seed=3), ti.mpo_xxz_nn(L, 0.5)
    res = {}
    for tol in (0.0, 1e-6):
        t = B.Tdvp(L, 2, 5, 8)
        t.set_params(eps=1e-10, krylov_tol=tol)
        t.set_mpo(W)
        t.set_mps(mps.psi, mps.lam)
        st = O.init_state(mps, W, O.Params(chi_max=8, eps=1e-10, krylov_tol=tol), p)
        for _ in range(3):
            t.step(0.05, p)
            O.step(st, 0.05)
        m = O.measure(st)
        assert t.chi() == O.chi_profile(st)
        assert np.abs(t.measure_sz() - m["sz"]).max() < 1e-6
        assert abs(t.measure_energy() - m["energy"]) < 1e-6
        res[tol] = t.measure_sz()
        t.close()
    assert np.abs(res[0.0] - res[1e-6]).max() < 1e-4


def test_svd_block_jacobi_forced_small(B):
    """The DMMA block-Jacobi SVD path (svd_bjac.cu, by default from 300
    columns) forced down to 32 columns (TDVP_SVD_BJ_MIN, read once per process,
    hence a subprocess): every SVD parity test above on ragged small shapes."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, TDVP_SVD_BJ_MIN="32")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-k", "svd and not forced",
                        os.path.abspath(__file__)], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


def test_svd_register_jacobi_forced_large(B):
    """The register-resident Jacobi (svd_rjac.cu) kept for every width up to
    1024 columns (TDVP_SVD_BJ_MIN = 1025, the segment-lane / U(1)-worker
    rule): every SVD parity test above, 300..1024 columns included."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, TDVP_SVD_BJ_MIN="1025")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-k", "svd and not forced",
                        os.path.abspath(__file__)], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


def test_svd_block_jacobi_forced_global_exchange(B):
    """The block Jacobi with its pair exchange through global memory (the
    fallback when the pair clusters cannot all be co-resident;
    TDVP_BJ_CLUSTER=0) forced down to 32 columns: every SVD parity test."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, TDVP_SVD_BJ_MIN="32", TDVP_BJ_CLUSTER="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-k", "svd and not forced",
                        os.path.abspath(__file__)], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
