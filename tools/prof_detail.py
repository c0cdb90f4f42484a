"""Per-phase kernel breakdown of one bench-family factorization (H2G_PROF_DETAIL
names GEMM/solve launches by phase; H2G_QR_DEBUG prints per-launch QR cycles)."""
import json
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2208_10907_b200 as h2
import os

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
warm = "--warm" in sys.argv  # one untimed factorization first (grown memory pool, as in bench.py)
xyz, q = h2.generate_points("sphere", n, 42)
MODE = os.environ.get("QR_MODE", "compressed")
COMPAT = os.environ.get("COMPAT", "0") == "1"
if warm:
    w = h2.Problem()
    w.set_kernel("yukawa", 1.0, 1.0, 1e-3)
    w.set_options(tol=1e-6, cap=100, qr_mode=MODE, reference_compat=COMPAT)
    w.build(xyz, q, 256)
    w.factor()
    w.close()
    print('=== main run', file=sys.stderr, flush=True)
p = h2.Problem()
p.set_kernel("yukawa", 1.0, 1.0, 1e-3)
p.set_options(tol=1e-6, cap=100, qr_mode=MODE, reference_compat=COMPAT)
p.set_profile(True)
p.build(xyz, q, 256)
p.factor()
ks = p.kernel_stats()
tot = sum(v["ms"] for v in ks.values())
for k, v in sorted(ks.items(), key=lambda kv: -kv[1]["ms"]):
    tf = v["flops"] / (v["ms"] * 1e-3) / 1e12 if v["ms"] else 0
    gb = v["bytes"] / (v["ms"] * 1e-3) / 1e9 if v["ms"] else 0
    print(f"{k:40s} {v['ms']:9.1f} ms {100*v['ms']/tot:5.1f}% n={v['launches']:5d} {tf:6.2f} TF/s {gb:8.1f} GB/s")
print(json.dumps(p.stats_dev()), json.dumps(p.phase_seconds()))
