"""Kernel microbenchmarks: H_eff^(2) matvec TFLOP/s over chi and D,
truncated-SVD time over matrix size.  Prints one JSON line per measurement.

python microbench.py [--heff] [--svd] [--chis 64,128,...] [--svd-n 64,...]
(TDVP_SVD_BW=4|8|16 forces the Jacobi block width.)
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--heff", action="store_true")
    ap.add_argument("--svd", action="store_true")
    ap.add_argument("--chis", default="64,128,256,512,1024")
    ap.add_argument("--svd-n", default="64,128,256,512,1024")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--svd-kind", default="gauss", choices=["gauss", "graded", "halfsmall"],
                    help="gauss: complex normal; graded: sigma_k = exp(-0.1 k); halfsmall: half O(1), half O(1e-2) "
                         "(the spectrum of the saturated bench two-site matrices)")
    a = ap.parse_args()
    import tdvp_inputs as ti
    from paper_1912_06127_b200 import tdvp as B
    if a.heff:
        Wnn = ti.mpo_xxz_nn(4, 0.5)[1]
        al, lam, _, _ = ti.fit_expsum(100, 9, 2.0)
        Wlr = ti.mpo_xxz_expsum(4, al, lam, 1.0)[1]
        for D, W in ((5, Wnn), (29, Wlr)):
            for chi in [int(x) for x in a.chis.split(",")]:
                if D == 29 and chi > 512:
                    continue
                ms, fl = B.bench_heff2(chi, W, W, reps=a.reps)
                print(json.dumps({"kernel": "heff2", "chi": chi, "D": D, "ms": ms, "tflops": fl / ms / 1e9}), flush=True)
    if a.svd:
        rng = np.random.default_rng(0)
        for n in [int(x) for x in a.svd_n.split(",")]:
            M = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
            if a.svd_kind != "gauss":
                q1, _ = np.linalg.qr(M)
                q2, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
                if a.svd_kind == "graded":
                    sv = np.exp(-0.1 * np.arange(n))
                else:
                    h = n // 2
                    sv = np.concatenate([np.sort(rng.uniform(0.5, 1.5, h))[::-1],
                                         1e-2 * np.sort(rng.uniform(0.0, 1.0, n - h))[::-1]])
                M = (q1 * sv[None, :]) @ q2.conj().T
            ms, sw = B.bench_svd(M, reps=3 if n >= 1024 else 5)
            print(json.dumps({"kernel": "svd", "n": n, "kind": a.svd_kind, "ms": ms,
                              "sweeps": sw}), flush=True)


if __name__ == "__main__":
    main()
