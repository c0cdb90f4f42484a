import os, sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2208_10907_b200 as h2
from oracle import cpu, ref
from paper_2208_10907_b200.pipeline import _fib_spheres
mode = os.environ.get("H2G_QR_MODE", "exact")
for geom, n, leaf, kind, cap, tol, st in [("cube", 4096, 128, "laplace", None, 1e-8, "h2"), ("cube", 4096, 128, "laplace", None, 1e-8, "hss"),
                                       ("sphere", 16384, 256, "yukawa", 100, 1e-6, "h2"), ("sphere", 65536, 256, "yukawa", 100, 1e-6, "h2")]:
    if geom == "cube":
        xyz, q = cpu.generate(geom, n, 42)
    else:
        xyz, q = _fib_spheres(n, 1, 3.0, 42)
    p = h2.Problem()
    p.set_kernel(kind, 1.0 if kind == "yukawa" else 0.0, 1.0, 1e-3)
    p.set_options(tol=tol, cap=cap, structure=st)
    p.build(xyz, q, leaf)
    t = time.time()
    try:
        p.factor()
    except h2.H2GError as e:
        print(mode, geom, n, st, "ERROR", e); continue
    tf = time.time() - t
    b = ref.splitmix_signed(n, 7)
    x = p.solve(b)
    r = np.linalg.norm(p.matvec(x) - b) / np.linalg.norm(b)
    ranks = [(l, int(rk.sum())) for l, rk in p.factor_levels()]
    print(mode, geom, n, st, "factor %.3f s dev %.3f" % (tf, p.stats_dev()["factor"]), "resid %.6e" % r, "ranks", ranks, "x[:3]", x[:3], flush=True)
    p.close()
