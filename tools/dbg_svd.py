"""Debug: svd_split vs numpy on assorted shapes; c1 chi profiles GPU vs oracle per step."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_06127_b200 as B
import tdvp_inputs as ti
from oracle import tdvp as O

rng = np.random.default_rng(1)
for (m, n) in [(2, 2), (2, 8), (8, 2), (4, 8), (8, 16), (16, 20), (20, 16), (16, 16), (20, 20), (32, 32), (4, 64), (64, 4), (40, 72), (72, 40), (256, 256), (128, 256), (256, 128), (512, 512), (300, 700)]:
    for kind in ("gauss", "graded", "rankdef"):
        A = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
        if kind == "graded":
            A = A * np.exp(-0.3 * np.arange(n))[None, :]
        if kind == "rankdef":
            r = max(1, min(m, n) // 3)
            A = A[:, :r] @ (rng.standard_normal((r, n)) + 1j * rng.standard_normal((r, n)))
        k = min(m, n)
        pl, S, pr, w = B.svd_split(A, k, eps=1e-12)
        s_ref = np.linalg.svd(A, compute_uv=False)
        chi_ref = int(np.sum(s_ref >= 1e-12 * s_ref[0]))
        rec = (pl / S[None, :]) @ pr
        P = rec
        U = pl / S[None, :]
        Wh = pr / S[:, None]
        print(f"{m}x{n} {kind:8s} chi {len(S)} ref {chi_ref} sig_err {np.abs(S - s_ref[:len(S)]).max() / s_ref[0]:.1e} "
              f"rec {np.linalg.norm(P - A) / np.linalg.norm(A):.1e} UU {np.abs(U.conj().T @ U - np.eye(len(S))).max():.1e} "
              f"WW {np.abs(Wh @ Wh.conj().T - np.eye(len(S))).max():.1e}", flush=True)

L, dt = 10, 0.05
mps, W = ti.neel_mps(L), ti.mpo_xxz_nn(L, 1.0)
for p in (1, 2):
    t = B.Tdvp(L, 2, 5, 32)
    t.set_params(eps=1e-12)
    t.set_mpo(W)
    t.set_mps(mps.psi, mps.lam)
    st = O.init_state(mps, W, O.Params(chi_max=32, eps=1e-12), p)
    for s in range(6):
        t.step(dt, p)
        O.step(st, dt)
        m_ = O.measure(st)
        print(p, s, t.chi(), O.chi_profile(st), np.abs(t.measure_sz() - m_["sz"]).max())
        _, glam = t.get_mps()
        _, olam = O.global_mps(st)
        for b, (a, o) in enumerate(zip(glam, olam)):
            if len(a) != len(o):
                print("   bond", b, "gpu tail", a[-3:] / a[0], "oracle tail", o[-3:] / o[0])
    t.close()
