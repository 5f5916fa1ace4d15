"""Run bench.py's workload for a few steps (for ncu launch lists and captures).

python tools/profile_step.py [workload] [steps]
Prints the library's launch count of every step, so an ncu launch list of the
same command can be cut to the last step (-s <launches before it>).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1912_06127_b200 as pkg  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5sat"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
wl = bench.workload_inputs(name)
t = pkg.Tdvp(wl["L"], 2, wl["D"], wl["chi"])
t.set_params(eps=wl["eps"])
t.set_mpo(wl["mpo"])
t.set_mps(wl["mps"].psi, wl["mps"].lam)
for k in range(steps):
    t.step(wl["dt"], 1)
    s = t.stats()
    print(f"step {k}: {s['step_ms']:.1f} ms, launches {s['kernel_launches']}, gemm {s['gemm_launches']}", flush=True)
t.close()
