"""p2TDVP hot-path benchmark (BASELINE.json metric).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c2sat|c5sat|...]

A "step" is one full 2TDVP/p2TDVP timestep (two half-sweeps: every pair
update = merge, K=8 Lanczos H_eff^(2) matvecs, SVD truncation, environment
update; every one-site backward update).  Default workload (N=1):
BASELINE configs[1] shapes (L=64 XXZ Delta=0.5, MPO D=5, chi_max=128,
eps=1e-10, dt=0.05) started from a seeded random inverse-canonical MPS with
saturated bonds so every timed step runs at chi=128.
value = device time per step (ms, lower is better), max over ranks.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# FP64 SIMT peak of B200: 64 DFMA/clk/SM (ncu sm__sass_thread_inst_executed_op_dfma_pred_on.peak_sustained)
# x 2 flop x 148 SMs x 1.965 GHz
FP64_ALU_PEAK_TF = 64 * 2 * 148 * 1.965e9 / 1e12
FP64_ALU_PEAK_SRC = ("derived: 64 DFMA/clk/SM (ncu dfma peak_sustained) x 2 x 148 SMs x 1.965 GHz "
                     "(clocks.max.sm); MEASURED_PEAKS.json has no FP64 entry")
METRIC = "2TDVP sweep time and H_eff complex-FP64 TFLOP/s (% of FP64 peak) at χ, 1/2/4/8 GPUs"

WORKLOADS = {
    # name: (L, Delta, chi_max, eps, dt, description)
    "c2sat": (64, 0.5, 128, 1e-10, 0.05,
              "configs[1] shapes: L=64 XXZ Delta=0.5 D=5 chi_max=128 eps=1e-10 dt=0.05, "
              "seeded random inverse-canonical MPS at saturated chi (SURVEY C6)"),
    "c3sat": (128, 1.5, 512, 1e-10, 0.02,
              "configs[2] shapes: L=128 XXZ Delta=1.5 D=5 chi_max=512 eps=1e-10 dt=0.02, saturated chi (C6)"),
    "c4sat": (100, 1.0, 256, 1e-12, 0.02,
              "configs[3] shapes: L=100 long-range XXZ J(r)~1/r^2 as 9 exponentials (MPO D=29) Delta=1 "
              "chi_max=256 eps=1e-12 dt=0.02, saturated chi (C6)"),
    "c5sat": (256, 1.0, 1024, 1e-12, 0.05,
              "configs[4] shapes: L=256 XXX D=5 chi_max=1024 eps=1e-12 dt=0.05, saturated chi (C6)"),
}


def jac_traffic():
    """DRAM bytes (read + write) per launch of the Jacobi kernel from the
    committed ncu --set full capture (profiles/r1b_traffic.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r1b_traffic.json")) as f:
            t = json.load(f)["rjac2"]
        return int(t["dram_bytes_read"]) + int(t["dram_bytes_write"])
    except (OSError, KeyError, ValueError):
        return None


def workload_inputs(name):
    import tdvp_inputs as ti
    L, Delta, chi, eps, dt, desc = WORKLOADS[name]
    if name == "c4sat":
        a, lam, _, _ = ti.fit_expsum(100, 9, 2.0)
        mpo = ti.mpo_xxz_expsum(L, a, lam, Delta)
    else:
        mpo = ti.mpo_xxz_nn(L, Delta)
    return dict(L=L, chi=chi, eps=eps, dt=dt, desc=desc, mpo=mpo, D=max(w.shape[3] for w in mpo),
                mps=ti.random_canonical_mps(L, chi, seed=2))


def mps_bytes(mps):
    return int(sum(p.nbytes for p in mps.psi) + sum(l.nbytes for l in mps.lam))


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- peaks
def fp64_peak_tflops():
    """Measured FP64 tensor peak: cuBLAS DGEMM 8192^3 and ZGEMM 4096^3 via torch
    (measurement only; not the product path), best of 5."""
    import torch
    best = {}
    for name, dt, n, fl in (("dgemm", torch.float64, 8192, 2.0), ("zgemm", torch.complex128, 4096, 8.0)):
        a = torch.randn(n, n, dtype=dt, device="cuda")
        b = torch.randn(n, n, dtype=dt, device="cuda")
        torch.matmul(a, b)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        best[name] = fl * n ** 3 / min(ts) / 1e12
        del a, b
    torch.cuda.empty_cache()
    return best


# ---------------------------------------------------------------- oracle (CPU baseline)
def cpu_baseline(wl, budget_s=12.0):
    """Time the oracle (as it stands) on a bounded sample of the same workload:
    bulk pair+single updates of the first half-sweep, scaled to a full step by
    the per-update contraction cost d chi_l chi_r (chi_l + chi_r)."""
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        threads = os.cpu_count()
    from oracle import tdvp as O
    L, dt = wl["L"], wl["dt"]
    st = O.init_state(wl["mps"], wl["mpo"], O.Params(chi_max=wl["chi"], eps=wl["eps"]), 1)
    seg = st.segs[0]
    chi = O.chi_profile(st)

    def w_pair(j):
        cl, cr = chi[j], chi[j + 2]
        return cl * cr * (cl + cr) * 2.0

    def w_back(j):
        cl, cr = chi[j], chi[j + 1]
        return cl * cr * (cl + cr)

    total_w = 2 * sum(w_pair(j) for j in range(L - 1)) + 2 * sum(w_back(j) for j in range(1, L - 1))
    t0 = time.perf_counter()
    done_w, n = 0.0, 0
    j = L // 2 - 4
    while time.perf_counter() - t0 < budget_s and j < L - 2:
        O._pair(st, seg, j, -0.5j * dt, True, False)
        O._back(st, seg, j + 1, dt)
        done_w += w_pair(j) + w_back(j + 1)
        n += 1
        j += 1
    el = time.perf_counter() - t0
    ms_step = el / done_w * total_w * 1e3
    return {"value": ms_step, "unit": "ms/step", "cores": int(threads), "kind": "oracle",
            "sample": f"{n} bulk pair+single updates (chi={wl['chi']}) of half-sweep 1 in {el:.1f} s, "
                      f"scaled to a full step by sum d*cl*cr*(cl+cr)"}


# ---------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2sat", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--lane-segments", type=int, default=8,
                    help="also time p2TDVP with this many segments as concurrent lanes on one GPU (N=1; 0 = off)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    wl = workload_inputs(args.workload)

    if args.impl == "reference":
        if rank != 0:
            return
        # the oracle is the reference arm for this tier: K bounded samples
        vals = []
        for _ in range(args.warmup):
            pass
        for _ in range(args.steps):
            vals.append(cpu_baseline(wl, budget_s=8.0))
        v = float(np.median([x["value"] for x in vals]))
        cb = dict(vals[0])
        cb["value"] = v
        print(json.dumps({"metric": METRIC, "value": v, "unit": "ms/step", "impl": "reference", "n_gpus": args.gpus,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False,
                          "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
                          "config": {"workload": args.workload, "desc": wl["desc"], "L": wl["L"],
                                     "chi_max": wl["chi"], "segments": 1},
                          "cpu_baseline": cb,
                          "e2e": {"value": v, "unit": "ms/step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return

    import torch
    import paper_1912_06127_b200 as pkg

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    p = world  # one segment per GPU; N=1 -> serial 2TDVP

    peaks = fp64_peak_tflops() if rank == 0 else {}

    L = wl["L"]
    t = pkg.Tdvp(L, 2, wl["D"], wl["chi"])
    t.set_params(eps=wl["eps"], timing=False)  # the timed steps run uninstrumented
    if world > 1:
        uid = [pkg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        t.comm_init(rank, world, uid[0])
    t.set_mpo(wl["mpo"])
    t.set_mps(wl["mps"].psi, wl["mps"].lam)
    dt = wl["dt"]
    for _ in range(args.warmup):
        t.step(dt, p)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    barrier()
    per = []
    with ClockSampler(local_rank) as clk:
        wall0 = time.perf_counter()
        for _ in range(args.steps):
            t.step(dt, p)
            per.append(t.stats())
        barrier()
        wall = time.perf_counter() - wall0
    step_ms = float(np.sum([s["step_ms"] for s in per]))
    if dist is not None:
        x = torch.tensor([step_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        step_ms = float(x.item())
    ms_per_step = step_ms / args.steps
    # breakdown pass: K more steps with CUDA events around every matvec, SVD,
    # Jacobi kernel and environment update (the events cost ~4% of a step,
    # so these steps are not the timed ones)
    t.set_params(eps=wl["eps"], timing=True)
    per_t = []
    for _ in range(args.steps):
        t.step(dt, p)
        per_t.append(t.stats())
    t.set_params(eps=wl["eps"], timing=False)
    bstep_ms = float(np.sum([s["step_ms"] for s in per_t]))
    per = per_t
    h2_ms = float(np.sum([s["heff2_ms"] for s in per]))
    h1_ms = float(np.sum([s["heff1_ms"] for s in per]))
    lz2_ms = float(np.sum([s["lanczos2_ms"] for s in per]))
    lz1_ms = float(np.sum([s["lanczos1_ms"] for s in per]))
    env_ms = float(np.sum([s["env_ms"] for s in per]))
    h2_fl = float(np.sum([s["heff2_flop"] for s in per]))
    svd_ms = float(np.sum([s["svd_ms"] for s in per]))
    jac_ms = float(np.sum([s["svd_jac_ms"] for s in per]))
    jac_fl = float(np.sum([s["svd_jac_flop"] for s in per]))
    sweeps = int(np.sum([s["svd_sweeps_total"] for s in per]))
    n_svd = int(np.sum([s["n_pair"] for s in per]))
    n_warm = int(np.sum([s["svd_warm"] for s in per]))
    launches = int(np.sum([s["kernel_launches"] for s in per]))
    gemm_launches = int(np.sum([s["gemm_launches"] for s in per]))

    # e2e: the same step through the C-ABI with HOST buffers (set_mps H2D incl.
    # the sequential environment build, step, get_mps D2H) every step
    e2e = None
    if not args.no_e2e and world == 1:
        mps = wl["mps"]
        t.step(dt, p)
        torch.cuda.synchronize()
        e0 = time.perf_counter()
        for _ in range(args.steps):
            t.set_mps(mps.psi, mps.lam)
            t.step(dt, p)
            psi, lam = t.get_mps()
        torch.cuda.synchronize()
        e_ms = (time.perf_counter() - e0) / args.steps * 1e3
        e2e = {"value": e_ms, "unit": "ms/step", "h2d_bytes_per_step": mps_bytes(mps),
               "d2h_bytes_per_step": int(sum(x.nbytes for x in psi) + sum(x.nbytes for x in lam))}
    # paper-mode Krylov (max 8 vectors, tolerance 1e-6; the
    # stopping rule runs on the device): a timing variant of the same step
    paper_mode = None
    if world == 1:
        t.set_params(eps=wl["eps"], timing=False, krylov_tol=1e-6)
        t.set_mps(wl["mps"].psi, wl["mps"].lam)
        for _ in range(args.warmup):
            t.step(dt, p)
        torch.cuda.synchronize()
        pms = []
        for _ in range(args.steps):
            t.step(dt, p)
            pms.append(t.stats()["step_ms"])
        t.set_params(eps=wl["eps"], timing=False)
        paper_mode = {"krylov_tol": 1e-6, "krylov_k_max": 8, "segments": p, "ms_per_step": float(np.mean(pms)),
                      "note": "timing variant; the headline value uses fixed K = 8 (parity mode, SURVEY AMB-5)"}

    # p2TDVP on this one GPU: P segments as concurrent lanes (own thread,
    # stream and workspace each), same workload, fresh state, same timing rules
    lanes = None
    if args.lane_segments > 1 and world == 1:
        q = args.lane_segments
        t.set_params(eps=wl["eps"], timing=False)
        t.set_mps(wl["mps"].psi, wl["mps"].lam)
        for _ in range(args.warmup):
            t.step(dt, q)
        torch.cuda.synchronize()
        lms, lfl = [], []
        for _ in range(args.steps):
            t.step(dt, q)
            st_ = t.stats()
            lms.append(st_["step_ms"])
            lfl.append(st_["svd_jac_flop"])
        lv = float(np.mean(lms))
        # all lanes' Jacobi work over the step time: how much of the FP64 ALU the
        # concurrent SVDs use together (the per-launch roofline above is one SVD)
        jagg = float(np.mean(lfl)) / (lv * 1e-3) / 1e12 if lv > 0 else None
        lanes = {"segments": q, "executor": "concurrent segment lanes on one GPU (thread + stream per segment)",
                 "partition": "uniform (PAPER.md:470)",
                 "ms_per_step": lv, "speedup_vs_serial": ms_per_step / lv if lv > 0 else None,
                 "jacobi_aggregate_tflops": jagg,
                 "jacobi_aggregate_frac_of_alu_peak": (jagg / FP64_ALU_PEAK_TF) if jagg else None}
        # the same with the chi-weighted partition (tdvp_partition_balanced)
        t.set_mps(wl["mps"].psi, wl["mps"].lam)
        bounds = pkg.balanced_partition(L, q, t.chi())
        t.set_partition(bounds)
        for _ in range(args.warmup):
            t.step(dt, q)
        torch.cuda.synchronize()
        bms = []
        for _ in range(args.steps):
            t.step(dt, q)
            bms.append(t.stats()["step_ms"])
        bv = float(np.mean(bms))
        t.set_partition(None)
        # strong scaling of p2TDVP on the one GPU (uniform partition, lanes)
        scal = []
        for qq in (2, 4, 16):
            if qq > L // 2:
                continue
            t.set_mps(wl["mps"].psi, wl["mps"].lam)
            for _ in range(max(1, args.warmup - 1)):
                t.step(dt, qq)
            torch.cuda.synchronize()
            sms = []
            for _ in range(args.steps):
                t.step(dt, qq)
                sms.append(t.stats()["step_ms"])
            scal.append({"segments": qq, "ms_per_step": float(np.mean(sms))})
        scal.append({"segments": q, "ms_per_step": lv})
        scal.sort(key=lambda x: x["segments"])
        lanes["balanced"] = {"bounds": bounds, "ms_per_step": bv,
                             "speedup_vs_serial": ms_per_step / bv if bv > 0 else None}
        lanes["scaling"] = [dict(x, speedup_vs_serial=ms_per_step / x["ms_per_step"]) for x in scal]
    t.close()

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    h2_tf = h2_fl / (h2_ms * 1e-3) / 1e12 if h2_ms > 0 else None
    zpeak = peaks.get("zgemm") if peaks else None
    jac_tf = jac_fl / (jac_ms * 1e-3) / 1e12 if jac_ms > 0 else None
    line = {
        "metric": METRIC, "value": ms_per_step, "unit": "ms/step", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": args.workload, "desc": wl["desc"], "L": L, "chi_max": wl["chi"], "D_mpo": wl["D"],
                   "segments": p, "parallelism": f"p2tdvp{p}" if p > 1 else "serial",
                   "l2": "working set (envs + MPS ~ 0.2 GB) larger than L2 (126 MB)"},
        # dominant kernel of the step: the Jacobi stage of the truncated SVD (FP64 SIMT, latency-bound)
        "roofline": {"kernel": "svd_rjac one-sided Jacobi (register-resident block pairs)", "bound": "alu",
                     "achieved": jac_tf, "peak": FP64_ALU_PEAK_TF, "unit": "TFLOP/s",
                     "frac": (jac_tf / FP64_ALU_PEAK_TF) if jac_tf else None, "traffic": jac_traffic(),
                     "peak_source": FP64_ALU_PEAK_SRC,
                     "flop_per_unit": "per sweep nc(nc-1)/2 * (16 mr + 24 (mr + nc)), sweeps counted on device",
                     "share_of_step": jac_ms / bstep_ms if bstep_ms > 0 else None,
                     "svd_calls": n_svd, "svd_warm_started": n_warm,
                     "sweeps_per_svd": sweeps / n_svd if n_svd else None},
        "heff2": {"kernel": "H_eff^(2) matvec (2 DMMA GEMMs + one fused sparse W_j W_{j+1} channel pass)", "bound": "tensor",
                  "achieved": h2_tf, "peak": zpeak, "unit": "TFLOP/s",
                  "frac": (h2_tf / zpeak) if (h2_tf and zpeak) else None,
                  "peak_source": f"measured in this run: cuBLAS FP64 {json.dumps(peaks)} (MEASURED_PEAKS.json has no FP64 entry)",
                  "share_of_step": h2_ms / bstep_ms if bstep_ms > 0 else None},
        "svd_share_of_step": svd_ms / bstep_ms if bstep_ms > 0 else None,
        "breakdown_ms_per_step_instrumented": bstep_ms / args.steps,
        "breakdown_ms_per_step": {"svd_total": svd_ms / args.steps, "svd_jacobi_kernel": jac_ms / args.steps,
                                  "lanczos2_total": lz2_ms / args.steps, "heff2_matvecs": h2_ms / args.steps,
                                  "lanczos1_total": lz1_ms / args.steps, "heff1_matvecs": h1_ms / args.steps,
                                  "env_updates": env_ms / args.steps,
                                  "rest": (bstep_ms - svd_ms - lz2_ms - lz1_ms - env_ms) / args.steps},
        "gpu_launches": launches,
        "gemm_launches": gemm_launches,
        "wall_s_timed": wall,
        "clocks": clk.summary(),
        "e2e": e2e,
        "p2tdvp_one_gpu": lanes,
        "paper_mode_krylov": paper_mode,
        "chi": wl["chi"],
    }
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(wl)
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
