import sys
import numpy as np
sys.path.insert(0, '.')
from oracle import ref
from paper_2208_10907_b200 import _lib as g


def beq(a, b):
    a = np.ascontiguousarray(a); b = np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.int64), b.view(np.int64))


rng = np.random.default_rng(0)
for (m, n, k) in [(5, 7, 3), (70, 130, 90), (150, 40, 300)]:
    a = rng.standard_normal((m, k)); b = rng.standard_normal((k, n)); c = rng.standard_normal((m, n))
    print('gemm', m, n, k, beq(g.gemm(a, b), ref.gemm(a, b)), beq(g.gemm(a, b, -1.0, c=c), ref.gemm(a, b, -1.0, c=c)),
          beq(g.gemm(a.T.copy(), b, transa=True), ref.gemm(a.T.copy(), b, transa=True)))
for n in [1, 7, 100, 170, 400]:
    a = rng.standard_normal((n, n)) + n * np.eye(n) * 0.1
    lg, pg = g.lu_factor(a); lr, pr = ref.lu_factor(a)
    print('lu', n, beq(lg, lr), np.array_equal(pg, pr), np.abs(lg - lr).max())
    for kind in ["solve", "lower", "upper", "transpose", "right", "upper_right"]:
        x = rng.standard_normal((n, 9)) if kind in ("solve", "lower", "upper", "transpose") else rng.standard_normal((9, n))
        xg = g.lu_solve(lr, pr, x, kind); xr = ref.lu_solve(lr, pr, x, kind)
        print('   ', kind, beq(xg, xr), np.abs(xg - xr).max())
for (dim, widths, tol, cap) in [(20, [5, 7, 3], 1e-8, None), (130, [100, 200, 50, 300], 1e-8, None), (130, [100, 200], 1e-4, 30)]:
    cols = []
    for w in widths:
        u = rng.standard_normal((dim, 6)); v = rng.standard_normal((6, w))
        cols.append(u @ v * np.exp(-np.arange(6))[None, :].T.sum() + 1e-6 * rng.standard_normal((dim, w)))
    concat = np.concatenate(cols, axis=1)
    offs = np.concatenate([[0], np.cumsum(widths)])
    qg, rg = g.basis_from_members(concat, offs, tol, cap); qr_, rr = ref.basis_from_members(concat, offs, tol, cap)
    print('basis', dim, rg, rr, beq(qg, qr_), np.abs(qg - qr_).max())
