"""N>1 host logic on CPU: world-size 2 and 4 gloo runs of the per-rank
schedule the NCCL path executes (libtdvp tdvp_plan) with real blocking
send/recv must (a) terminate (no deadlock) and (b) reproduce the sequential
BSP oracle exactly (SURVEY App. A "Independence")."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import tdvp_inputs as ti
from oracle import tdvp as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,L", [(2, 10), (4, 12)])
def test_gloo_protocol_matches_sequential_oracle(tmp_path, world, L):
    steps, dt = 2, 0.05
    out = str(tmp_path / "dist.npz")
    port = free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   T_L=str(L), T_STEPS=str(steps), T_DT=str(dt), T_OUT=out, OMP_NUM_THREADS="1",
                   OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "_dist_worker.py")], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
    for p in procs:
        try:
            p.wait(timeout=240)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            pytest.fail("distributed protocol deadlocked")
        assert p.returncode == 0, p.stdout.read().decode()[-3000:]
    got = np.load(out)
    a, lam, _, _ = ti.fit_expsum(50, 3, 2.0)
    W = ti.mpo_xxz_expsum(L, a, lam, 0.8)
    st = O.init_state(ti.bloch_mps(L, 0), W, O.Params(chi_max=16, eps=1e-12), world)
    for _ in range(steps):
        O.step(st, dt)
    psi, lams = O.global_mps(st)
    for j in range(L):
        assert got[f"psi{j}"].shape == psi[j].shape
        assert np.allclose(got[f"psi{j}"], psi[j], atol=1e-13, rtol=0)
    for b in range(L - 1):
        assert np.allclose(got[f"lam{b}"], lams[b], atol=1e-13, rtol=0)
