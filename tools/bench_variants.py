"""The other BASELINE.json geometries / kernels at the largest size this
algorithm holds on one B200 (N = 65,536; its pieces are O(N^2)):
device-timed build + factor + solve (1 warm-up, 2 timed steps, compressed QR,
corrected assembly, fill-absorption abort disabled), residual against the
matrix-free direct sum. One JSON line per variant.

  python tools/bench_variants.py [N]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_10907_b200 as h2  # noqa: E402
from oracle import ref  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
VARIANTS = [
    dict(name="c2_fibonacci_sphere_yukawa (the bench)", geometry="sphere", kernel="yukawa", alpha=1.0, cap=100),
    dict(name="c2_uniform_iid_sphere_yukawa (BASELINE's wording)", geometry="uniform_sphere", kernel="yukawa",
         alpha=1.0, cap=100),
    dict(name="c4_family_cube_laplace_cap128", geometry="cube", kernel="laplace", alpha=0.0, cap=128),
    dict(name="c5_family_ellipsoids64_laplace_cap128", geometry="ellipsoids", kernel="laplace", alpha=0.0, cap=128,
         spheres=64),
]
for v in VARIANTS:
    try:
        xyz, q = h2.generate_points(v["geometry"], N, 42, v.get("spheres", 1))
        b = ref.splitmix_signed(N, 7)
        p = h2.Problem()
        p.set_kernel(v["kernel"], v["alpha"], 1.0, 1e-3)
        p.set_options(tol=1e-6, cap=v["cap"], qr_mode="compressed", reference_compat=False,
                      abort_residual_factor=1e30)

        def step():
            p.build(xyz, q, 256)
            p.factor()
            return p.solve(b)

        step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(2):
            x = step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 2
        sd = p.stats_dev()
        r = float(np.linalg.norm(p.matvec(x) - b) / np.linalg.norm(b))
        line = dict(v, n=N, ms_per_step=ms, points_per_s=N / (ms * 1e-3), factor_s=sd["factor"], levels=p.levels,
                    rank_sums=[[int(l), int(np.sum(rk)), int(np.max(rk))] for l, rk in p.factor_levels()],
                    solve_rel_residual=r, max_fill_residual=p.max_fill_residual(),
                    timing="host-buffer C ABI calls (H2D/D2H inside), torch CUDA events on the default stream")
        p.close()
    except Exception as e:
        line = dict(v, n=N, error=str(e)[:300])
    print(json.dumps(line), flush=True)
