"""Write the oracle's results for the large-chi parity cases (tests/golden/).

Calls ONLY oracle/ (and the seeded input generators in tdvp_inputs/); nothing
here touches the CUDA path.  The GPU tests (tests/test_gpu_large_chi.py)
rebuild the same seeded inputs, check them against the stored input
fingerprint, run the library and compare with these stored oracle outputs,
so the slow CPU oracle at chi = 1024 does not run on the GPU box.

python tools/make_goldens.py [case ...]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import tdvp_inputs as ti  # noqa: E402
from oracle import tdvp as O  # noqa: E402

# name: (L, chi_max, eps, dt, steps, segment counts, MPO, description)
CASES = {
    # configs[3] shapes: long-range 1/r^2 as 9 exponentials (MPO D = 29), chi_max = 256 binding
    "sat256_lr": (20, 256, 1e-12, 0.02, 2, (1, 2), "lr", "L=20 long-range XXX (D=29) chi_max=256 eps=1e-12 dt=0.02"),
    # configs[2] shapes: XXZ Delta = 1.5, chi_max = 512 binding
    "sat512": (20, 512, 1e-10, 0.02, 2, (1, 2), "xxz1.5", "L=20 XXZ Delta=1.5 (D=5) chi_max=512 eps=1e-10 dt=0.02"),
    # configs[4] shapes: XXX, chi_max = 1024 binding at the centre bond (2048 x 2048 SVD)
    "sat1024": (22, 1024, 1e-12, 0.05, 1, (1, 2), "xxx", "L=22 XXX (D=5) chi_max=1024 eps=1e-12 dt=0.05"),
}


def case_inputs(name):
    L, chi, eps, dt, steps, ps, model, desc = CASES[name]
    if model == "lr":
        a, lam, _, _ = ti.fit_expsum(100, 9, 2.0)
        W = ti.mpo_xxz_expsum(L, a, lam, 1.0)
    elif model == "xxz1.5":
        W = ti.mpo_xxz_nn(L, 1.5)
    else:
        W = ti.mpo_xxz_nn(L, 1.0)
    mps = ti.random_canonical_mps(L, chi, seed=2)
    return dict(L=L, chi=chi, eps=eps, dt=dt, steps=steps, ps=ps, W=W, mps=mps, desc=desc)


def fingerprint(mps):
    """Input fingerprint: Frobenius norms of Psi_j and the first Schmidt value of
    each bond (detects a changed input generator, not a CUDA quantity)."""
    return np.array([np.linalg.norm(p) for p in mps.psi] + [float(l[0]) for l in mps.lam] +
                    [float(np.abs(p).sum()) for p in mps.psi])


def run(name):
    c = case_inputs(name)
    out = {"fingerprint": fingerprint(c["mps"])}
    meta = {"desc": c["desc"], "steps": c["steps"], "ps": list(c["ps"])}
    for p in c["ps"]:
        t0 = time.time()
        st = O.init_state(c["mps"], c["W"], O.Params(chi_max=c["chi"], eps=c["eps"]), p)
        for _ in range(c["steps"]):
            O.step(st, c["dt"])
        m = O.measure(st)
        _, lam = O.global_mps(st)
        out[f"p{p}_sz"] = np.asarray(m["sz"])
        out[f"p{p}_energy"] = np.array([m["energy"]])
        out[f"p{p}_norm"] = np.array([m["norm"]])
        out[f"p{p}_chi"] = np.array(O.chi_profile(st))
        out[f"p{p}_trunc"] = np.array([int(st.stats.trunc_active)])
        for b, l in enumerate(lam):
            out[f"p{p}_lam{b}"] = np.asarray(l)
        meta[f"p{p}_seconds"] = time.time() - t0
        print(name, p, f"{time.time() - t0:.1f} s", "chi", O.chi_profile(st), flush=True)
    path = os.path.join(ROOT, "tests", "golden", f"{name}.npz")
    np.savez_compressed(path, meta=np.array(json.dumps(meta)), **out)


if __name__ == "__main__":
    for n in (sys.argv[1:] or list(CASES)):
        run(n)
