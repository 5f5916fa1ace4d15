"""CPU ORACLE for the p2TDVP hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg may import this package.  The product path
(paper_1912_06127_b200, libtdvp.so) never imports, links or executes it,
and this package never imports the product.  The only shared code is the
seeded input generator module ``tdvp_inputs`` (no method arithmetic).

Plain, slow, obviously-correct NumPy/SciPy complex128 implementation of
serial 2TDVP and the segment-parallel p2TDVP of Secular et al.,
arXiv:1912.06127, executed step by step in the paper's order.
Pins: tests/test_oracle_*.py.
"""
from .tdvp import (  # noqa: F401
    Params, State, env_left, env_right, apply_h1, apply_h2, merge_theta,
    svd_truncate, expm_lanczos, init_state, step, measure, to_dense,
    serial_step_literal, plan_partition, directions,
)
