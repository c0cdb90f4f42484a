"""Gaussian kernel (BASELINE configs[2], not in the reference): exp(-r^2/0.1)
+ 1e-2 I on points uniform in the unit cube, leaf 256, cap 128. Factor + solve
through the GPU path; residual by the matrix-free direct sum; kernel blocks vs
the C oracle.  usage: python tools/dev_gaussian.py N [N ...] [--mode M] [--tol T]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_10907_b200 as h2  # noqa: E402
from oracle import cpu  # noqa: E402

args = sys.argv[1:]
mode = "compressed"
tol = 1e-6
leaf = 256
if "--mode" in args:
    i = args.index("--mode"); mode = args[i + 1]; del args[i:i + 2]
if "--tol" in args:
    i = args.index("--tol"); tol = float(args[i + 1]); del args[i:i + 2]
if "--leaf" in args:
    i = args.index("--leaf"); leaf = int(args[i + 1]); del args[i:i + 2]
for n in map(int, args):
    xyz, q = cpu.generate("cube", n, 42)
    b = np.random.default_rng(7).uniform(-1, 1, n)
    p = h2.Problem()
    p.set_kernel("gaussian", 10.0, 1.0, 1e-2)
    p.set_options(tol=tol, cap=128, qr_mode=mode)
    p.build(xyz, q, leaf)
    p.factor()
    x = p.solve(b)
    r = float(np.linalg.norm(p.matvec(x) - b) / np.linalg.norm(b))
    sd = p.stats_dev()
    print(json.dumps({"n": n, "mode": mode, "tol": tol, "leaf": leaf, "levels": p.levels, "resid": r,
                      "ranks": [int(rk.sum()) for _, rk in p.factor_levels()], "factor_s": sd["factor"],
                      "build_s": sd["build"]}), flush=True)
    p.close()
