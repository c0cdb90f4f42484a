"""Factorization time and points/s vs N on the bench workload family (sphere,
Yukawa, leaf 256, cap 100, tol 1e-6): one JSON line per N, device-timed
(CUDA events) after one warm-up factorization at that N; with --ref N_MAX the
unmodified reference (oracle/_ref, all host cores) runs the same inputs up to
N_MAX."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_10907_b200 as h2  # noqa: E402
from paper_2208_10907_b200.pipeline import _fib_spheres  # noqa: E402

argv = sys.argv[1:]
ref_max = 0
if "--ref" in argv:
    i = argv.index("--ref")
    ref_max = int(argv[i + 1])
    del argv[i:i + 2]
args = argv
for n in map(int, args):
    xyz, q = _fib_spheres(n, 1, 3.0, 42)
    b = np.random.default_rng(7).uniform(-1, 1, n)

    def run():
        p = h2.Problem()
        p.set_kernel("yukawa", 1.0, 1.0, 1e-3)
        p.set_options(tol=1e-6, cap=100)
        p.set_profile(True)
        p.build(xyz, q, 256)
        p.factor()
        x = p.solve(b)
        return p, x

    p, _ = run()
    p.close()
    p, x = run()
    sd = p.stats_dev()
    ks = p.kernel_stats()
    resid = float(np.linalg.norm(p.matvec(x) - b) / np.linalg.norm(b))
    qr = ks.get("qr", {"ms": 0, "bytes": 0})
    line = {"n": n, "levels": p.levels, "build_s": sd["build"], "factor_s": sd["factor"],
            "solve_s": sd["solve"], "factor_points_per_s": n / sd["factor"],
            "step_points_per_s": n / (sd["build"] + sd["factor"] + sd["solve"]),
            "qr_share": qr["ms"] * 1e-3 / sd["factor"], "qr_gbs": qr["bytes"] / max(qr["ms"], 1e-9) / 1e6,
            "residual": resid}
    p.close()
    if n <= ref_max:
        from oracle import ref
        cfg = ref.make_config(256, tol=1e-6, cap=100, kernel="yukawa", alpha_m=1.0, reg=1e-3, scale=1.0,
                              threads=os.cpu_count() or 1)
        xr, qr_ = ref.generate("sphere", n, 42)
        r = ref.RefRun(xr, qr_, cfg)
        t0 = time.perf_counter()
        r.build().factor()
        r.solve(b)
        line["ref_step_s"] = time.perf_counter() - t0
        line["ref_cores"] = os.cpu_count()
    print(json.dumps(line), flush=True)
