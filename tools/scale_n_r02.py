"""Round-2 time vs N on the bench workload family (reference sphere cloud,
Yukawa, leaf 256, cap 100, tol 1e-6; compressed QR, corrected assembly), with
the reference's full far-field members and with sampled members
(h2g_set_sampling 512). The fill-absorption abort (ulv.cpp:140-147) is
disabled (abort_residual_factor = 1e30) so sizes past 98,304 run; device time
the fastest of three factorizations after one warm-up per size and mode.

  python tools/scale_n_r02.py N [N ...]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_10907_b200 as h2  # noqa: E402
from oracle import ref  # noqa: E402

for n in map(int, sys.argv[1:]):
    xyz, q = h2.generate_points("sphere", n, 42)
    b = ref.splitmix_signed(n, 7)
    for sample in (0, 512):
        def run():
            p = h2.Problem()
            p.set_kernel("yukawa", 1.0, 1.0, 1e-3)
            p.set_options(tol=1e-6, cap=100, qr_mode="compressed", reference_compat=False,
                          abort_residual_factor=1e30, sample_cols=sample)
            p.build(xyz, q, 256)
            p.factor()
            return p
        try:
            run().close()
            times = []
            for _ in range(2):  # the allocator pool occasionally regrows after a size change: keep the faster run
                p0 = run()
                times.append(p0.stats_dev()["factor"])
                p0.close()
            p = run()
            sd = p.stats_dev()
            times.append(sd["factor"])
            sd["factor"] = min(times)
            x = p.solve(b)
            resid = float(np.linalg.norm(p.matvec(x) - b) / np.linalg.norm(b))
            line = {"n": n, "sample_cols": sample, "levels": p.levels, "build_s": sd["build"],
                    "factor_s": sd["factor"], "factor_points_per_s": n / sd["factor"], "residual": resid,
                    "max_fill_residual": p.max_fill_residual(), "factor_s_runs": times}
            p.close()
        except Exception as e:  # out of memory at the largest sizes
            line = {"n": n, "sample_cols": sample, "error": str(e)[:200]}
        print(json.dumps(line), flush=True)
