"""Run the UNMODIFIED reference once at the benched config and commit its result.

TEST INFRASTRUCTURE (development container only; /root/reference is needed to
build oracle/_ref*). BASELINE configs[1] as benched: N points of the reference's
Fibonacci-lattice unit sphere (geometry.cpp:64-95, seed 42), Yukawa
exp(-r)/(r + 1e-3) (scale 1), leaf 256, eta 1, cap 100, tol 1e-6, h2/nodep,
b = SplitMix64(7).next_signed() (report.cpp solve_rhs convention).

Writes tests/golden/c2_<N>[_<tag>].json (+ .npz with x): wall times per phase,
peak RSS, ranks per factorized level, cutoff dims, hashes of points / perm / x.

  H2REF_LIB=oracle/_ref_native/libh2ref.so python tools/ref_pin_c2.py 65536 native
  FIXED=1 python tools/ref_pin_c2.py 65536 fixed      # corrected reference (oracle/_ref_fixed)
"""
import json
import os
import resource
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from oracle import ref  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    tag = sys.argv[2] if len(sys.argv) > 2 else ""
    threads = int(os.environ.get("THREADS", os.cpu_count() or 1))
    fixed = os.environ.get("FIXED") == "1"  # the corrected build (oracle/fix_reference.py)
    xyz, q = ref.generate("sphere", n, 42)
    cfg = ref.make_config(256, tol=1e-6, cap=100, kernel="yukawa", alpha_m=1.0, reg=1e-3,
                          scale=1.0, threads=threads)
    r = ref.RefRun(xyz, q, cfg, fixed=fixed)
    t0 = time.perf_counter()
    r.build()
    t1 = time.perf_counter()
    r.factor()
    t2 = time.perf_counter()
    b = ref.splitmix_signed(n, 7)
    x = r.solve(b)
    t3 = time.perf_counter()
    levels = [(lvl, ranks.tolist()) for lvl, ranks in r.factor_levels()]
    cut_lvl, cut_dims = r.cutoff()
    st = r.stats()
    out = {
        "what": ("corrected reference (oracle/_ref_fixed, fix_reference.py)" if fixed else
                 "unmodified reference (oracle/_ref*)") + ", benched config C2",
        "lib": (ref.FIXED_PATH if fixed else ref.LIB_PATH).replace(os.path.dirname(HERE) + "/", ""),
        "n": n, "leaf": 256, "tol": 1e-6, "cap": 100, "kernel": "yukawa", "alpha_m": 1.0,
        "reg": 1e-3, "scale": 1.0, "geometry": "sphere(1) seed 42", "b": "splitmix_signed(n, 7)",
        "threads": threads, "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": "),
        "wall_build_s": t1 - t0, "wall_factor_s": t2 - t1, "wall_solve_s": t3 - t2,
        "peak_rss_gb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6,
        "stats": st,
        "levels": levels, "cutoff_level": int(cut_lvl), "cutoff_dims": cut_dims.tolist(),
        "points_fnv": "%016x" % ref.fnv64(xyz.view(np.int64).ravel()),
        "perm_fnv": "%016x" % ref.fnv64(r.perm()),
        "x_fnv": "%016x" % ref.fnv64(x.view(np.int64)),
        "max_fill_residual": r.max_fill_residual(),
    }
    base = os.path.join(os.path.dirname(HERE), "tests", "golden", f"c2_{n}" + (f"_{tag}" if tag else ""))
    np.savez_compressed(base + ".npz", x=x)
    with open(base + ".json", "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "levels"}, indent=1))


if __name__ == "__main__":
    main()
