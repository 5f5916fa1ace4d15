"""GPU: the diagnostics of SURVEY.md §8(f) N2 through the C-ABI.

* tdvp_overlap / infidelity I = 1 - |<a|b>| / sqrt(<a|a><b|b>) (PAPER.md,
  benchmark section: serial vs parallel states) against the dense inner
  product of the two downloaded states (oracle.to_dense, L <= 12).
* tdvp_reorthonormalize: the physical state is unchanged
  (up to normalisation), the new Lambda_j are the exact Schmidt values of the
  dense state, every Psi_j is an orthogonality centre again, and a serial
  untruncated run continues identically.
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


def handle(B, W, mps, chi_max, eps=1e-12):
    D = max(max(w.shape[0] for w in W), max(w.shape[3] for w in W))
    t = B.Tdvp(len(W), 2, D, chi_max)
    t.set_params(eps=eps)
    t.set_mpo(W)
    t.set_mps(mps.psi, mps.lam)
    return t


def dense(t):
    psi, lam = t.get_mps()
    return O.to_dense(psi, lam)


def schmidt(v, L, b):
    """Schmidt values across bond b (sites 0..b | b+1..L-1) of a dense state."""
    return np.linalg.svd(v.reshape(2 ** (b + 1), -1), compute_uv=False)


def test_overlap_matches_dense(B):
    L = 10
    W = ti.mpo_xxz_nn(L, 0.5)
    a = handle(B, W, ti.random_canonical_mps(L, 8, seed=4), 16)
    b = handle(B, W, ti.random_canonical_mps(L, 8, seed=5), 16)
    b.step(0.05, 2)
    va, vb = dense(a), dense(b)
    o = a.overlap(b)
    ref = np.vdot(va, vb)
    assert abs(o - ref) < 1e-12 * max(1.0, abs(ref))
    assert abs(b.overlap(a) - np.conj(ref)) < 1e-12 * max(1.0, abs(ref))
    assert abs(a.overlap(a) - a.measure_norm()) < 1e-12
    assert abs(a.infidelity(a)) < 1e-13
    a.close()
    b.close()


def test_infidelity_serial_vs_parallel(B):
    """Untruncated: p = 1 and p = 4 reach the same state (infidelity at
    rounding level); truncated: the GPU infidelity equals the one of the
    oracle's serial and parallel runs (both tiny here: the two schedules
    truncate at chi = 8 in different orders, I ~ 1e-13)."""
    L = 12
    W = ti.mpo_xxz_nn(L, 0.5)
    s = handle(B, W, ti.neel_mps(L), 64)
    p = handle(B, W, ti.neel_mps(L), 64)
    for _ in range(6):
        s.step(0.05, 1)
        p.step(0.05, 4)
    assert s.infidelity(p) < 1e-12
    s.close()
    p.close()

    mps = ti.random_canonical_mps(L, 8, seed=2)
    s = handle(B, W, mps, 8, eps=1e-10)
    p = handle(B, W, mps, 8, eps=1e-10)
    sts, stp = (O.init_state(mps, W, O.Params(chi_max=8, eps=1e-10), q) for q in (1, 2))
    for _ in range(3):
        s.step(0.05, 1)
        p.step(0.05, 2)
        O.step(sts, 0.05)
        O.step(stp, 0.05)
    va, vb = (O.to_dense(*O.global_mps(x)) for x in (sts, stp))
    ref = 1 - abs(np.vdot(va, vb)) / np.sqrt(np.vdot(va, va).real * np.vdot(vb, vb).real)
    got = s.infidelity(p)
    assert abs(got - ref) < 1e-9 + 1e-2 * ref
    s.close()
    p.close()


def test_reorthonormalize_gauge(B):
    """A chain whose Lambda_j are NOT its Schmidt values (perturbed) is
    re-gauged: same physical state, exact Schmidt values, canonical Psi_j."""
    L = 10
    rng = np.random.default_rng(11)
    mps = ti.random_canonical_mps(L, 8, seed=6)
    lam = [l * np.exp(0.3 * rng.standard_normal(l.shape)) for l in mps.lam]
    W = ti.mpo_xxz_nn(L, 0.5)
    D = max(max(w.shape[0] for w in W), max(w.shape[3] for w in W))
    t = B.Tdvp(L, 2, D, 16)
    t.set_mpo(W)
    t.set_mps(mps.psi, lam)
    v0 = O.to_dense(mps.psi, lam)
    v0 = v0 / np.linalg.norm(v0)
    t.reorthonormalize()
    psi, lam2 = t.get_mps()
    v1 = O.to_dense(psi, lam2)
    assert abs(t.measure_norm() - 1.0) < 1e-12
    assert np.abs(v1 - v0).max() < 1e-12  # no phase freedom: the gauge change is exact
    for b in range(L - 1):
        s = schmidt(v0, L, b)
        k = len(lam2[b])
        assert k == np.count_nonzero(s > 1e-14 * s[0])
        assert np.allclose(lam2[b], s[:k], rtol=1e-11, atol=1e-14)
    # every Psi_j an orthogonality centre: sum |Psi_j|^2 = 1
    for j in range(L):
        assert abs(np.linalg.norm(psi[j]) - 1.0) < 1e-12
    t.close()


def test_reorthonormalize_continues_run(B):
    """Untruncated run (p = 2): reorthonormalising mid-run does not change
    the trajectory beyond rounding (the Lambda_j are already Schmidt values)."""
    L = 10
    W = ti.mpo_xxz_nn(L, 0.5)
    a = handle(B, W, ti.neel_mps(L), 64)
    b = handle(B, W, ti.neel_mps(L), 64)
    for n in range(6):
        a.step(0.05, 2)
        b.step(0.05, 2)
        if n == 2:
            b.reorthonormalize()
    assert np.abs(a.measure_sz() - b.measure_sz()).max() < 1e-10
    assert abs(a.measure_energy() - b.measure_energy()) < 1e-10
    assert a.infidelity(b) < 1e-12
    a.close()
    b.close()


def test_many_lanes_match_oracle(B):
    """16 concurrent segment lanes (L = 32, 2 sites each) against the oracle on
    the same partition; then the round-robin executor gives identical numbers."""
    import os
    L, p = 32, 16
    mps, W = ti.random_canonical_mps(L, 8, seed=8), ti.mpo_xxz_nn(L, 0.5)
    st = O.init_state(mps, W, O.Params(chi_max=8, eps=1e-10), p)
    for _ in range(2):
        O.step(st, 0.05)
    m = O.measure(st)
    out = {}
    for lanes in ("1", "0"):
        os.environ["TDVP_LANES"] = lanes
        try:
            t = handle(B, W, mps, 8, eps=1e-10)
        finally:
            os.environ.pop("TDVP_LANES", None)
        for _ in range(2):
            t.step(0.05, p)
        assert t.chi() == O.chi_profile(st)
        out[lanes] = t.measure_sz()
        assert np.abs(out[lanes] - m["sz"]).max() < 1e-6
        t.close()
    assert np.array_equal(out["1"], out["0"])  # same kernels, same order per segment: bit-identical


def test_maybe_reorthonormalize(B):
    L = 10
    W = ti.mpo_xxz_nn(L, 0.5)
    t = handle(B, W, ti.random_canonical_mps(L, 8, seed=6), 16)
    assert not t.maybe_reorthonormalize(1e-3)  # canonical input: norm 1
    psi, lam = t.get_mps()
    t.set_mps([2.0 * x if j == 3 else x for j, x in enumerate(psi)], lam)  # norm 4
    assert t.maybe_reorthonormalize(1e-3)
    assert abs(t.measure_norm() - 1.0) < 1e-12
    t.close()


def test_set_partition_validation(B):
    L = 16
    t = handle(B, ti.mpo_xxz_nn(L, 0.5), ti.neel_mps(L), 8)
    for bad in ([(0, 0), (1, 15)],                      # segment of one site
                [(1, 7), (8, 15)],                      # does not start at 0
                [(0, 3), (4, 9), (10, 15)],             # odd p
                [(0, 7), (8, 8)] + [(9, 15)]):          # odd p, short segment
        with pytest.raises(B.TdvpError) as e:
            t.set_partition(bad)
        assert e.value.code in (-1, -3)
    t.set_partition([(0, 3), (4, 15)])
    t.step(0.05, 2)   # uses the explicit partition
    t.step(0.05, 4)   # p differs: the uniform rule
    t.set_partition(None)
    t.step(0.05, 2)
    assert abs(t.measure_norm() - 1.0) < 1e-9
    t.close()


def test_set_get_mps_pinned_buffers(B):
    """set_mps from page-locked host arrays, get_mps into caller-owned pinned
    buffers (the bench's e2e path): same state as the default allocating
    get_mps after a step, buffers filled in place; mismatched out buffers
    fall back to fresh arrays; a non-finite entry is rejected (the threaded
    validation) and the handle keeps its state."""
    import torch
    L, chi_max = 12, 16
    W = ti.mpo_xxz_nn(L, 0.7)
    mps = ti.random_canonical_mps(L, chi_max, seed=11)

    def pin(a):
        x = torch.empty(a.shape, dtype=torch.complex128 if np.iscomplexobj(a) else torch.float64,
                        pin_memory=True).numpy()
        x[...] = a
        return x

    t = handle(B, W, mps, chi_max, eps=1e-14)
    t.set_mps([pin(x) for x in mps.psi], [pin(x) for x in mps.lam])
    t.step(0.05, 2)
    ref_psi, ref_lam = t.get_mps()
    chi = t.chi()
    out = ([pin(np.zeros((chi[j], 2, chi[j + 1]), np.complex128)) for j in range(L)],
           [pin(np.zeros(chi[b + 1])) for b in range(L - 1)])
    psi, lam = t.get_mps(out)
    assert all(a is b for a, b in zip(psi, out[0])) and all(a is b for a, b in zip(lam, out[1]))
    for a, b in zip(psi, ref_psi):
        assert np.array_equal(a, b)
    for a, b in zip(lam, ref_lam):
        assert np.array_equal(a, b)
    bad = ([np.zeros((1, 2, 1), np.complex128)] * L, out[1])
    psi2, _ = t.get_mps(bad)
    assert psi2[0] is not bad[0] and all(np.array_equal(a, b) for a, b in zip(psi2, ref_psi))
    # non-finite input: rejected, the evolved state is kept
    nf = [x.copy() for x in ref_psi]
    nf[L // 2].flat[-1] = np.nan
    with pytest.raises(B.TdvpError):
        t.set_mps(nf, ref_lam)
    psi3, _ = t.get_mps()
    assert all(np.array_equal(a, b) for a, b in zip(psi3, ref_psi))
    t.close()
