"""Lanczos vector-pass GB/s and H_eff^(2) TF/s per chi bin for one workload
(timing=1 steps): python tools/lz_bins.py [workload] [steps]"""
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
t.set_params(eps=wl["eps"], timing=True)
t.set_mpo(wl["mpo"])
t.set_mps(wl["mps"].psi, wl["mps"].lam)
t.step(wl["dt"], 1)
for k in range(steps):
    t.step(wl["dt"], 1)
    s = t.stats()
    row = []
    for b in range(4):
        ms, by = s["lz_ms_bin"][b], s["lz_bytes_bin"][b]
        hm, hf = s["heff2_ms_bin"][b], s["heff2_flop_bin"][b]
        if ms > 0:
            row.append(f"bin{b}: lz {ms:.2f} ms {by / ms / 1e6:.0f} GB/s | h2 {hm:.1f} ms {hf / hm / 1e9 if hm else 0:.1f} TF/s")
    print(f"step {k}: {s['step_ms']:.1f} ms; " + "; ".join(row), flush=True)
t.close()
