"""Front half (tree + admissibility lists + near-field arena, Pipeline::build)
at the BASELINE configs the O(N^2) exact-member factorization cannot reach on
one GPU: C3 N = 262,144 cube, C4 N = 1,048,576 cube (Laplace, diag 1e3), C5
N = 4,194,304 on 64 random ellipsoids. Device time (CUDA events) of a second
build after a warm-up one; one JSON line per config."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2208_10907_b200 as h2  # noqa: E402
from paper_2208_10907_b200.pipeline import generate_ellipsoids, generate_uniform_cube  # noqa: E402

CONFIGS = [("c3_cube262144", "cube", 262144), ("c4_cube1048576", "cube", 1048576),
           ("c5_ellipsoids4194304", "ellipsoids", 4194304)]
for name, geom, n in CONFIGS:
    xyz, q = generate_uniform_cube(n, 42) if geom == "cube" else generate_ellipsoids(n, 64, 42)
    for rep in range(2):
        p = h2.Problem()
        p.set_kernel("laplace", 0.0, 1.0, 1e-3)
        p.set_options(tol=1e-6, cap=128)
        t0 = time.perf_counter()
        p.build(xyz, q, 256)
        wall = time.perf_counter() - t0
        if rep == 1:
            near = [int(p.L.h2g_list_count(p.h, p.levels, 0)), int(p.L.h2g_list_count(p.h, p.levels, 1))]
            entries = int(p.L.h2g_near_entries(p.h))
            st = p.stats()
            dev = p.stats_dev()["build"]
            print(json.dumps({"config": name, "n": n, "levels": p.levels, "leaf_near_pairs": near[0],
                              "leaf_far_pairs": near[1], "near_field_entries": entries,
                              "near_field_gb": entries * 8 / 1e9, "build_dev_s": dev, "build_wall_s": wall,
                              "points_per_s": n / dev, "near_field_write_gbs": entries * 8 / dev / 1e9,
                              "t_tree_s": st["t_tree"], "t_classify_s": st["t_classify"],
                              "t_near_s": st["t_near"]}), flush=True)
        p.close()
