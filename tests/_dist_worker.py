"""One rank of the CPU (gloo) message-passing check of the p2TDVP protocol.

Each rank executes libtdvp's own per-rank op list (tdvp_plan, the schedule the
NCCL path runs) with the oracle's local updates and REAL blocking gloo
send/recv between neighbours.  Rank 0 gathers the owner copies and writes
them to an .npz for the test to compare with the sequential BSP oracle.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import tdvp_inputs as ti  # noqa: E402
from oracle import tdvp as O  # noqa: E402
from paper_1912_06127_b200 import tdvp as B  # noqa: E402


def send_arrays(arrs, peer):
    for a in arrs:
        a = np.ascontiguousarray(a)
        cplx = np.iscomplexobj(a)
        hdr = torch.tensor([a.ndim, int(cplx)] + list(a.shape) + [0] * (4 - a.ndim), dtype=torch.int64)
        dist.send(hdr, peer)
        flat = a.view(np.float64).reshape(-1) if cplx else a.astype(np.float64).reshape(-1)
        dist.send(torch.from_numpy(flat.copy()), peer)


def recv_arrays(n, peer):
    out = []
    for _ in range(n):
        hdr = torch.zeros(6, dtype=torch.int64)
        dist.recv(hdr, peer)
        nd, cplx = int(hdr[0]), int(hdr[1])
        shape = [int(x) for x in hdr[2:2 + nd]]
        size = int(np.prod(shape)) * (2 if cplx else 1)
        buf = torch.zeros(size, dtype=torch.float64)
        dist.recv(buf, peer)
        a = buf.numpy()
        out.append(a.view(np.complex128).reshape(shape).copy() if cplx else a.reshape(shape).copy())
    return out


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    L, steps, dt, chi = int(os.environ["T_L"]), int(os.environ["T_STEPS"]), float(os.environ["T_DT"]), 16
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, lam, _, _ = ti.fit_expsum(50, 3, 2.0)
    W = ti.mpo_xxz_expsum(L, a, lam, 0.8)
    st = O.init_state(ti.bloch_mps(L, 0), W, O.Params(chi_max=chi, eps=1e-12), world)
    seg = st.segs[rank]
    s, e = seg.s, seg.e
    for _ in range(steps):
        for h in (1, 2):
            for kind, j, full, build in B.plan(L, world, h, rank):
                if kind == 1:
                    O._pair(st, seg, j, (-1.0j if full else -0.5j) * dt, bool(build & 1), bool(build & 2))
                elif kind == 2:
                    O._back(st, seg, j, dt)
                elif kind == 3:
                    send_arrays([seg.psi[e + 1], seg.lam[e], seg.beta[e + 1]], rank + 1)
                elif kind == 4:
                    seg.psi[s], seg.lam[s - 1], seg.beta[s] = recv_arrays(3, rank - 1)
                elif kind == 5:
                    send_arrays([seg.psi[s], seg.gamma[s]], rank - 1)
                elif kind == 6:
                    seg.psi[e + 1], seg.gamma[e + 1] = recv_arrays(2, rank + 1)
    owned = {"psi": {j: seg.psi[j] for j in range(s, e + 1)},
             "lam": {b: seg.lam[b] for b in range(s, min(e, L - 2) + 1)}}
    got = [None] * world if rank == 0 else None
    dist.gather_object(owned, got, dst=0)
    if rank == 0:
        out = {}
        for o in got:
            for j, x in o["psi"].items():
                out[f"psi{j}"] = x
            for b, x in o["lam"].items():
                out[f"lam{b}"] = x
        np.savez(os.environ["T_OUT"], **out)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
