"""Corrected assembly vs N on the bench family (sphere, Yukawa, leaf 256, cap
100, tol 1e-6): residual and device time per QR mode. GPU only.

  python tools/corrected_scale.py 16384 32768 65536
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2208_10907_b200 as h2  # noqa: E402
from paper_2208_10907_b200.pipeline import splitmix_signed  # noqa: E402


def main():
    cap = int(os.environ.get("CAP", "100"))
    tol = float(os.environ.get("TOL", "1e-6"))
    modes = os.environ.get("MODES", "exact,compressed").split(",")
    compats = [c == "1" for c in os.environ.get("COMPAT", "0").split(",")]
    for n in map(int, sys.argv[1:]):
        xyz, q = h2.generate_points("sphere", n, 42)
        b = splitmix_signed(n, 7)
        for compat in compats:
            for mode in modes:
                p = h2.Problem()
                p.set_kernel("yukawa", 1.0, 1.0, 1e-3)
                p.set_options(tol=tol, cap=cap or None, qr_mode=mode, reference_compat=compat)
                t0 = time.perf_counter()
                try:
                    p.build(xyz, q, 256)
                    p.factor()
                    x = p.solve(b)
                except Exception as e:  # noqa: BLE001
                    print(json.dumps({"n": n, "mode": mode, "compat": compat, "error": str(e)}), flush=True)
                    p.close()
                    continue
                dt = time.perf_counter() - t0
                r = float(np.linalg.norm(p.matvec(x) - b) / np.linalg.norm(b))
                lv = [(int(l), int(rk.sum()), int(rk.max())) for l, rk in p.factor_levels()]
                sd = p.stats_dev()
                print(json.dumps({"n": n, "mode": mode, "compat": compat, "cap": cap, "tol": tol,
                                  "residual": r, "wall_s": dt, "factor_dev_s": sd["factor"],
                                  "levels": lv, "max_fill_residual": p.max_fill_residual()}), flush=True)
                p.close()


if __name__ == "__main__":
    main()
