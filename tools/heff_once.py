"""Time one H_eff^(2) matvec (DMMA GEMMs + channel mix) at chi_L = chi_R = chi
with the XXX D = 5 MPO: python tools/heff_once.py chi [reps] -> (ms, TFLOP/s)"""
import sys

sys.path.insert(0, '.')
import tdvp_inputs as ti  # noqa: E402
from paper_1912_06127_b200 import tdvp as B  # noqa: E402

chi = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
W = ti.mpo_xxz_nn(8, 1.0)
print(chi, B.bench_heff2(chi, W[3], W[4], reps=reps))
