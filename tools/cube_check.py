import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2208_10907_b200 as h2
from oracle import ref
for n, leaf in ((8192, 128), (8192, 256), (16384, 256)):
    xyz, q = h2.generate_points("cube", n, 42)
    b = ref.splitmix_signed(n, 7)
    for tol in (1e-6, 1e-8, 1e-10):
        for compat in (True, False):
            p = h2.Problem()
            p.set_kernel("laplace", 0.0, 1.0, 1e-3)
            p.set_options(tol=tol, cap=None, qr_mode="blocked", reference_compat=compat, abort_residual_factor=1e30)
            p.build(xyz, q, leaf)
            try:
                p.factor()
                x = p.solve(b)
                r = float(np.linalg.norm(p.matvec(x) - b) / np.linalg.norm(b))
                print(n, leaf, tol, "compat" if compat else "corrected", "resid %.3e" % r, [int(np.max(rk)) for _, rk in p.factor_levels()], "fill %.1e" % p.max_fill_residual(), flush=True)
            except Exception as e:
                print(n, leaf, tol, compat, "ERR", str(e)[:80], flush=True)
            p.close()
