"""Step time of p2TDVP with p segments on ONE GPU: concurrent segment lanes
(default) vs the single-stream round-robin executor (TDVP_LANES=0).
python tools/lanes_bench.py [workload] [p ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1912_06127_b200 as pkg  # noqa: E402

wl = bench.workload_inputs(sys.argv[1] if len(sys.argv) > 1 else "c2sat")
ps = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
for p in ps:
    t = pkg.Tdvp(wl["L"], 2, 5, wl["chi"])
    t.set_params(eps=wl["eps"], timing=bool(int(os.environ.get("LB_TIMING", "0"))),
                 krylov_tol=float(os.environ.get("LB_KTOL", "0")))
    t.set_mpo(wl["mpo"])
    t.set_mps(wl["mps"].psi, wl["mps"].lam)
    if os.environ.get("LB_BAL") and p > 1:
        t.set_partition(pkg.balanced_partition(wl["L"], p, t.chi()))
    for _ in range(2):
        t.step(wl["dt"], p)
    ms = []
    w0 = time.perf_counter()
    for _ in range(3):
        t.step(wl["dt"], p)
        ms.append(t.stats()["step_ms"])
    wall = (time.perf_counter() - w0) / 3 * 1e3
    st = t.stats()
    print(f"p={p} lanes={os.environ.get('TDVP_LANES', '1')} step_ms={np.mean(ms):.1f} wall_ms={wall:.1f} "
          f"E={t.measure_energy():.12f} chi_max={max(t.chi())} n_pair={st['n_pair']}", flush=True)
    if os.environ.get("LB_TIMING"):
        print("   summed over lanes: " + " ".join(f"{k}={st[k]:.1f}" for k in
              ("svd_ms", "svd_jac_ms", "lanczos2_ms", "heff2_ms", "lanczos1_ms", "heff1_ms", "env_ms")), flush=True)
    t.close()
