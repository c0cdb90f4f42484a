"""Scale probe: exact-member GPU factorization on the bench workload family."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_2208_10907_b200 as h2
from paper_2208_10907_b200.pipeline import _fib_spheres, generate_uniform_cube

for n, leaf, geom in [(int(a), int(b), c) for a, b, c in (x.split(':') for x in sys.argv[1:])]:
    xyz, q = _fib_spheres(n, 1, 3.0, 42) if geom == 'sphere' else generate_uniform_cube(n, 42)
    p = h2.Problem()
    p.set_kernel('yukawa', 1.0, 1.0, 1e-3)
    p.set_options(tol=float(__import__('os').environ.get('TOL', '1e-6')), cap=100)
    warm = int(__import__('os').environ.get('WARM', '0'))
    try:
        for _ in range(warm):  # grow the device memory pool before the measured run
            pw = h2.Problem()
            pw.set_kernel('yukawa', 1.0, 1.0, 1e-3)
            pw.set_options(tol=float(__import__('os').environ.get('TOL', '1e-6')), cap=100)
            pw.build(xyz, q, leaf)
            pw.factor()
            pw.close()
    except h2.H2GError as e:
        print(n, leaf, geom, 'factor error:', e, flush=True)
        continue
    p.set_profile(True)
    t = time.time(); p.build(xyz, q, leaf); tb = time.time() - t
    t = time.time()
    try:
        p.factor()
    except h2.H2GError as e:
        print(n, leaf, geom, 'factor error:', e, flush=True)
        continue
    tf = time.time() - t
    b = np.random.default_rng(7).uniform(-1, 1, n)
    t = time.time(); x = p.solve(b); ts = time.time() - t
    y = p.matvec(x)
    print(n, leaf, geom, 'build %.3f factor %.3f solve %.3f' % (tb, tf, ts), 'dev', p.stats_dev(),
          'resid %.3e' % (np.linalg.norm(y - b) / np.linalg.norm(b)), flush=True)
    print('   levels', [(l, int(r.max()), float(r.mean())) for l, r in p.factor_levels()], p.cutoff())
    ks = p.kernel_stats()
    for k, v in sorted(ks.items(), key=lambda kv: -kv[1]['ms']):
        print('   %-6s %9.1f ms %6d launches %10.3e flops %10.3e bytes  %.1f GB/s %.2f TF/s' % (
            k, v['ms'], v['launches'], v['flops'], v['bytes'], v['bytes'] / v['ms'] / 1e6 if v['ms'] else 0,
            v['flops'] / v['ms'] / 1e9 if v['ms'] else 0))
    print('   stats', p.stats(), flush=True)
    print('   phases', p.phase_seconds(), flush=True)
    p.close()
