import sys
import numpy as np
sys.path.insert(0, '.')
from oracle import ref
from paper_2208_10907_b200 import _lib as g
def beq(a, b): return np.array_equal(np.ascontiguousarray(a).view(np.int64), np.ascontiguousarray(b).view(np.int64))
rng = np.random.default_rng(5)
for n in [64, 100, 200, 257]:
    a = rng.standard_normal((n, n)) + 0.1 * n * np.eye(n)
    lu, perm = ref.lu_factor(a)
    for kind in ["solve", "lower", "upper"]:
        for cols in [48, 300]:
            x = rng.standard_normal((n, cols))
            print(n, kind, cols, beq(g.lu_solve(lu, perm, x, kind), ref.lu_solve(lu, perm, x, kind)))
