"""Single large GEMMs through h2g_gemm (time the gemm_kernel launches with ncu)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2208_10907_b200 import _lib as g
rng = np.random.default_rng(0)
for (m, n, k) in [(128, 8192, 4096), (100, 8192, 4096), (2048, 2048, 2048), (256, 256, 256)]:
    a = rng.standard_normal((m, k)); b = rng.standard_normal((k, n))
    c = g.gemm(a, b)
    print(m, n, k, 'ok', flush=True)
