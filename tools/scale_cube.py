"""BASELINE configs[3] family at growing N: points uniform in the unit cube
(SplitMix64 seed 42), Laplace 1/(r + 1e-3) (diagonal 1e3), leaf 256, eta 1,
cap 128, tol 1e-6 (env TOL), compressed QR mode. One JSON line per N (device time,
after one warm-up at 65,536); stops at the first N that fails and prints why.
usage: python tools/scale_cube.py N [N ...]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_10907_b200 as h2  # noqa: E402
from oracle import cpu  # noqa: E402


def run(n, prof=False):
    xyz, q = cpu.generate("cube", n, 42)
    b = np.random.default_rng(7).uniform(-1, 1, n)
    p = h2.Problem()
    p.set_kernel("laplace", 0.0, 1.0, 1e-3)
    p.set_options(tol=float(os.environ.get("TOL", "1e-6")), cap=128, qr_mode="compressed")
    p.build(xyz, q, 256)
    p.factor()
    x = p.solve(b)
    r = float(np.linalg.norm(p.matvec(x) - b) / np.linalg.norm(b))
    sd = p.stats_dev()
    out = {"n": n, "levels": p.levels, "build_s": sd["build"], "factor_s": sd["factor"],
           "solve_s": sd["solve"], "factor_points_per_s": n / sd["factor"], "residual": r,
           "ranks": [int(rk.sum()) for _, rk in p.factor_levels()]}
    p.close()
    return out


run(16384)
for n in map(int, sys.argv[1:]):
    try:
        print(json.dumps(run(n)), flush=True)
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"n": n, "error": str(e)}), flush=True)
        break
