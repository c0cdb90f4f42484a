"""One build+factor+solve of the bench workload family at a profiling size."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2208_10907_b200 as h2

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
xyz, q = h2.generate_points("sphere", n, 42)
p = h2.Problem()
p.set_kernel("yukawa", 1.0, 1.0, 1e-3)
import os
p.set_options(tol=1e-6, cap=100, qr_mem_budget=int(float(os.environ.get("QR_BUDGET", "0"))))
p.build(xyz, q, 256)
p.factor()
x = p.solve(np.random.default_rng(7).uniform(-1, 1, n))
print("ok", n, p.stats_dev())
