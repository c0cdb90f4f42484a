"""Golden fixtures of the CORRECTED reference (oracle/_ref_fixed/libh2ref.so:
the unmodified reference sources with the three covered-coupling fixes of
oracle/fix_reference.py applied at build time). They pin the GPU path's
reference_compat = 0 mode. Run here, commit the output:

    make -C oracle ref-fixed && python tests/golden/make_golden_fixed.py

Writes tests/golden/fixed.json: per case the ranks per factorized level,
cutoff dims, FNV of x for b = SplitMix64(7), and the relative residual
||A x - b|| / ||b|| from the reference's own dense matvec (solve.cpp:234-239)
next to the unmodified reference's residual on the same system.
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle import ref  # noqa: E402

CASES = [
    # name, geometry, n, leaf, tol, cap, kernel, structure, spheres
    ("cube1024", "cube", 1024, 128, 1e-8, None, "laplace", "h2", 1),
    ("cube2048", "cube", 2048, 128, 1e-8, None, "laplace", "h2", 1),
    ("c1_cube4096", "cube", 4096, 128, 1e-8, None, "laplace", "h2", 1),
    ("cube4096_tol1e-6", "cube", 4096, 128, 1e-6, None, "laplace", "h2", 1),
    ("spheres8_4096", "sphere", 4096, 128, 1e-6, None, "laplace", "h2", 8),
    ("sphere4096_yukawa_cap100_tol1e-6_leaf256", "sphere", 4096, 256, 1e-6, 100, "yukawa", "h2", 1),
    ("sphere8192_yukawa_cap100_tol1e-6_leaf256", "sphere", 8192, 256, 1e-6, 100, "yukawa", "h2", 1),
    ("hss1024", "cube", 1024, 128, 1e-8, None, "laplace", "hss", 1),
]


def fbits(a):
    return ref.fnv64(np.ascontiguousarray(a, dtype=np.float64).view(np.int64).ravel())


def main():
    out = {"generator": "oracle/_ref_fixed/libh2ref.so (reference proj/src + oracle/fix_reference.py, "
                        "-O3 -mavx2 -mfma)", "cases": {}}
    for name, geom, n, leaf, tol, cap, kernel, structure, spheres in CASES:
        xyz, q = ref.generate(geom, n, 42, spheres)
        cfg = ref.make_config(leaf, tol=tol, cap=cap, kernel=kernel, structure=structure, reg=1e-3,
                              scale=1.0, alpha_m=1.0)
        b = ref.splitmix_signed(n, 7)
        rec = dict(geometry=geom, n=n, leaf=leaf, tol=tol, cap=cap, kernel=kernel,
                   structure=structure, spheres=spheres)
        for fixed in (True, False):
            r = ref.RefRun(xyz, q, cfg, fixed=fixed).build()
            t0 = time.perf_counter()
            r.factor()
            dt = time.perf_counter() - t0
            x = r.solve(b)
            res = float(np.linalg.norm(r.dense_matvec(x) - b) / np.linalg.norm(b))
            if fixed:
                rec["ranks"] = {str(l): rk.tolist() for l, rk in r.factor_levels()}
                lvl, dims = r.cutoff()
                rec["cutoff"] = [int(lvl), dims.tolist()]
                rec["x_fnv"] = fbits(x)
                rec["residual"] = res
                rec["factor_s"] = dt
            else:
                rec["residual_unmodified_reference"] = res
        out["cases"][name] = rec
        print(name, "residual %.3e (unmodified %.3e)" % (rec["residual"], rec["residual_unmodified_reference"]),
              flush=True)
    with open(os.path.join(HERE, "fixed.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
