import numpy as np, sys
sys.path.insert(0, '.')
from paper_1912_06127_b200 import tdvp as B
rng = np.random.default_rng(0)
n = int(sys.argv[1])
M = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
print(B.bench_svd(M, reps=1))
