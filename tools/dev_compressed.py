"""Compressed QR mode (qr_mode = 2) vs the exact and blocked modes: solve
residual, per-level rank sums and device factor time, on the golden cases and
on the bench workload family (sphere, Yukawa, leaf 256, cap 100, tol 1e-6).

usage: python tools/dev_compressed.py [golden] [N ...]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_10907_b200 as h2  # noqa: E402
from oracle import cpu, ref  # noqa: E402
from paper_2208_10907_b200.pipeline import _fib_spheres  # noqa: E402


def run(xyz, q, b, kernel, opts, leaf, mode, prof=False):
    p = h2.Problem()
    p.set_kernel(*kernel)
    p.set_options(qr_mode=mode, **opts)
    p.set_profile(prof)
    p.build(xyz, q, leaf)
    p.factor()
    x = p.solve(b)
    r = float(np.linalg.norm(p.matvec(x) - b) / np.linalg.norm(b))
    sd = p.stats_dev()
    ranks = [int(rk.sum()) for _, rk in p.factor_levels()]
    ks = p.kernel_stats() if prof else {}
    p.close()
    return {"mode": mode, "resid": r, "ranks": ranks, "factor_s": sd["factor"],
            "kernels": {k: round(v["ms"], 1) for k, v in ks.items()}}, x


def golden_cases():
    g = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "golden.json")))
    for name, rec in g["cases"].items():
        if "residual" not in rec:
            continue
        xyz, q = cpu.generate(rec["geometry"], rec["n"], 42, rec["spheres"])
        b = ref.splitmix_signed(rec["n"], 7)
        kind = rec["kernel"]
        kernel = (kind, 1.0 if kind == "yukawa" else 0.0, rec["scale"], rec["reg"])
        opts = dict(tol=rec["tol"], cap=rec["cap"], structure=rec["structure"])
        out = {"case": name, "ref_resid": rec["residual"], "tol": rec["tol"]}
        xs = {}
        for mode in ("exact", "compressed"):
            out[mode], xs[mode] = run(xyz, q, b, kernel, opts, rec["leaf"], mode)
        out["x_rel_diff"] = float(np.linalg.norm(xs["compressed"] - xs["exact"]) / np.linalg.norm(xs["exact"]))
        print(json.dumps(out), flush=True)


def bench_family(n):
    xyz, q = _fib_spheres(n, 1, 3.0, 42)
    b = np.random.default_rng(7).uniform(-1, 1, n)
    kernel = ("yukawa", 1.0, 1.0, 1e-3)
    opts = dict(tol=1e-6, cap=100)
    for mode in ("blocked", "compressed"):
        run(xyz, q, b, kernel, opts, 256, mode)  # warm-up
        out, _ = run(xyz, q, b, kernel, opts, 256, mode, prof=True)
        out["n"] = n
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for a in sys.argv[1:]:
        if a == "golden":
            golden_cases()
        else:
            bench_family(int(a))
