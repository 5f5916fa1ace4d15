"""Time the library's truncated-SVD path on a seeded complex Gaussian matrix.

python tools/svd_once.py n [reps]   -> (ms per SVD, Jacobi sweeps)
"""
import sys

import numpy as np

sys.path.insert(0, '.')
from paper_1912_06127_b200 import tdvp as B  # noqa: E402

rng = np.random.default_rng(0)
n = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
M = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
print(B.bench_svd(M, reps=reps))
