"""Developer parity sweep: B200 path vs the compiled reference (oracle/_ref)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from oracle import ref
import paper_2208_10907_b200 as h2


def bits_equal(a, b):
    a = np.ascontiguousarray(a); b = np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.int64), b.view(np.int64))


def run(geom, n, leaf, tol=1e-8, cap=None, kernel="laplace", reg=1e-3, scale=1.0, structure="h2", seed=42):
    xyz, q = ref.generate(geom, n, seed)
    cfg = ref.make_config(leaf, tol=tol, cap=cap, kernel=kernel, reg=reg, scale=scale, structure=structure)
    t = time.time(); R = ref.RefRun(xyz, q, cfg).build().factor(); tr = time.time() - t
    G = h2.Problem()
    G.set_kernel(kernel, 1.0 if kernel == "yukawa" else 0.0, scale, reg)
    G.set_options(tol=tol, cap=cap, structure=structure)
    t = time.time(); G.build(xyz, q, leaf); tb = time.time() - t
    t = time.time(); G.factor(); tf = time.time() - t
    out = {}
    out['perm'] = np.array_equal(G.perm(), R.perm())
    beG, geoG = G.nodes(); beR, geoR = R.nodes()
    out['nodes'] = np.array_equal(beG, beR) and bits_equal(geoG, geoR)
    ok = True
    for l in range(1, R.levels + 1):
        for far in (0, 1):
            a = G.lists(l, far); b = R.lists(l, far)
            ok &= np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    out['lists'] = ok
    out['near'] = bits_equal(G.leaf_dense(), R.leaf_dense())
    fg = G.factor_levels(); fr = R.factor_levels()
    out['ranks'] = len(fg) == len(fr) and all(a[0] == b[0] and np.array_equal(a[1], b[1]) for a, b in zip(fg, fr))
    if not out['ranks']:
        for a, b in zip(fg, fr):
            print('   lvl', a[0], b[0], 'gpu', a[1][:16], 'ref', b[1][:16])
    out['cutoff'] = G.cutoff()[0] == R.cutoff()[0] and np.array_equal(G.cutoff()[1], R.cutoff()[1])
    # bases at leaf
    L = R.levels
    bok = True
    maxd = 0
    for k in range(1 << L):
        for side in (0, 1):
            a, ra = G.basis(L, k, side); b, rb = R.basis(L, k, side)
            bok &= bits_equal(a, b)
            if a.shape == b.shape: maxd = max(maxd, np.abs(a - b).max())
    out['leaf_bases_bitwise'] = bok
    out['leaf_bases_maxdiff'] = maxd
    if out['cutoff']:
        tg = G.top(); tr_ = R.top()
        out['top_bitwise'] = bits_equal(tg[0], tr_[0]) and np.array_equal(tg[1], tr_[1])
        if tg[0].shape == tr_[0].shape:
            out['top_maxrel'] = np.abs(tg[0] - tr_[0]).max() / np.abs(tr_[0]).max()
    b = ref.splitmix_signed(n, 7)
    t = time.time(); xg = G.solve(b); ts = time.time() - t
    xr = R.solve(b)
    out['x_bitwise'] = bits_equal(xg, xr)
    out['x_rel'] = np.linalg.norm(xg - xr) / np.linalg.norm(xr)
    yg = G.matvec(xg)
    out['resid_gpu'] = np.linalg.norm(yg - b) / np.linalg.norm(b)
    if n <= 4096:
        yr = R.dense_matvec(xr)
        out['resid_ref'] = np.linalg.norm(yr - b) / np.linalg.norm(b)
        out['matvec_bitwise'] = bits_equal(R.dense_matvec(xg), yg)
    out['t_ref_factor'] = tr; out['t_gpu_build'] = tb; out['t_gpu_factor'] = tf; out['t_gpu_solve'] = ts
    print(geom, n, leaf, tol, cap, kernel, structure, out, flush=True)
    return out


if __name__ == '__main__':
    run('cube', 512, 64)
    run('cube', 1024, 128)
    run('cube', 1024, 128, structure='hss')
    run('cube', 2048, 128)
    run('sphere', 2048, 128, kernel='yukawa', cap=100)
    run('cube', 4096, 128)
