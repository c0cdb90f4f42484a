"""Sampled far-field basis members (h2g_set_sampling) against the reference's
full members: factor time, per-level rank sums, solve residual and the
distance of x from the unsampled run, on the bench workload family.

  python tools/sample_study.py N [sample_cols ...]
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, '.')
import paper_2208_10907_b200 as h2  # noqa: E402
from oracle import ref  # noqa: E402


def run(xyz, q, b, sample, mode="compressed", compat=False, tol=1e-6, cap=100):
    p = h2.Problem()
    p.set_kernel("yukawa", 1.0, 1.0, 1e-3)
    p.set_options(tol=tol, cap=cap, qr_mode=mode, reference_compat=compat, sample_cols=sample)
    p.build(xyz, q, 256)
    t0 = time.perf_counter()
    p.factor()
    wall = time.perf_counter() - t0
    dev = p.stats_dev()
    x = p.solve(b)
    r = float(np.linalg.norm(p.matvec(x) - b) / np.linalg.norm(b))
    levels = [[int(l), int(np.sum(rk)), int(np.max(rk))] for l, rk in p.factor_levels()]
    out = dict(sample_cols=sample, residual=r, wall_s=wall, factor_dev_s=dev.get("factor"), levels=levels,
               max_fill_residual=p.max_fill_residual())
    p.close()
    return out, x


def main():
    n = int(sys.argv[1])
    samples = [int(a) for a in sys.argv[2:]] or [0, 1024, 512, 256, 128]
    xyz, q = h2.generate_points("sphere", n, 42)
    b = ref.splitmix_signed(n, 7)
    run(xyz, q, b, 0)  # warm the memory pool
    x0 = None
    for sc in samples:
        out, x = run(xyz, q, b, sc)
        if sc == 0:
            x0 = x
        if x0 is not None:
            out["x_rel_diff_vs_full"] = float(np.linalg.norm(x - x0) / np.linalg.norm(x0))
        out["n"] = n
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
