"""Time the parts of the bench's e2e step (set_mps / step / get_mps) on c2sat."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1912_06127_b200 as pkg
wl = bench.workload_inputs("c2sat")
t = pkg.Tdvp(wl["L"], 2, 5, wl["chi"])
t.set_params(eps=wl["eps"])
t.set_mpo(wl["mpo"])
mps = wl["mps"]
t.set_mps(mps.psi, mps.lam)
t.step(wl["dt"], 1)
acc = {"set_mps": 0.0, "step": 0.0, "get_mps": 0.0}
for _ in range(3):
    torch.cuda.synchronize()
    a = time.perf_counter(); t.set_mps(mps.psi, mps.lam); b = time.perf_counter()
    t.step(wl["dt"], 1); c = time.perf_counter()
    psi, lam = t.get_mps(); d = time.perf_counter()
    acc["set_mps"] += b - a; acc["step"] += c - b; acc["get_mps"] += d - c
print({k: round(v / 3 * 1e3, 2) for k, v in acc.items()}, "step_ms(device)", t.stats()["step_ms"])
