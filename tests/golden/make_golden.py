"""Generate golden fixtures from the UNMODIFIED reference (oracle/_ref/libh2ref.so,
compiled from /root/reference by oracle/Makefile). Run here, commit the output:

    python tests/golden/make_golden.py

Writes tests/golden/golden.json (hashes, ranks, residuals) and golden.npz
(solutions x for small cases, primitive-kernel inputs/outputs).
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle import ref  # noqa: E402

CASES = [
    # name, geometry, n, leaf, tol, cap, kernel, structure, reg, scale, spheres
    ("cube512", "cube", 512, 64, 1e-8, None, "laplace", "h2", 1e-3, 1.0, 1),
    ("cube1024", "cube", 1024, 128, 1e-8, None, "laplace", "h2", 1e-3, 1.0, 1),
    ("cube1024_default_kernel", "cube", 1024, 128, 1e-8, None, "laplace", "h2", None, 4 * np.pi, 1),
    ("hss1024", "cube", 1024, 128, 1e-8, None, "laplace", "hss", 1e-3, 1.0, 1),
    ("cube2048", "cube", 2048, 128, 1e-8, None, "laplace", "h2", 1e-3, 1.0, 1),
    ("sphere2048_yukawa_cap100", "sphere", 2048, 128, 1e-8, 100, "yukawa", "h2", 1e-3, 1.0, 1),
    ("line1024", "line", 1024, 64, 1e-8, None, "laplace", "h2", 1e-3, 1.0, 1),
    ("spheres8_4096", "sphere", 4096, 128, 1e-6, None, "laplace", "h2", 1e-3, 1.0, 8),
    ("c1_cube4096", "cube", 4096, 128, 1e-8, None, "laplace", "h2", 1e-3, 1.0, 1),
    ("sphere4096_yukawa_cap100_tol1e-6_leaf256", "sphere", 4096, 256, 1e-6, 100, "yukawa", "h2", 1e-3, 1.0, 1),
]
STRUCTURE_ONLY = [
    ("c2_sphere65536", "sphere", 65536, 256, 1),
    ("cube262144", "cube", 262144, 256, 1),
]


def fbits(a):
    return ref.fnv64(np.ascontiguousarray(a, dtype=np.float64).view(np.int64).ravel())


def structure_record(r):
    be, geo = r.nodes()
    rec = {"levels": r.levels, "perm_fnv": ref.fnv64(r.perm()), "nodes_fnv": ref.fnv64(be.ravel()),
           "geo_fnv": fbits(geo), "lists": {}}
    for lvl in range(1, r.levels + 1):
        npt, nid = r.lists(lvl, 0)
        fpt, fid = r.lists(lvl, 1)
        rec["lists"][str(lvl)] = [ref.fnv64(npt), ref.fnv64(nid), ref.fnv64(fpt), ref.fnv64(fid),
                                  int(len(nid)), int(len(fid))]
    return rec


def main():
    out = {"generator": "oracle/_ref/libh2ref.so (reference proj/src, -O3 -mavx2 -mfma)", "cases": {}}
    arrays = {}
    for name, geom, n, leaf, tol, cap, kernel, structure, reg, scale, spheres in CASES:
        xyz, q = ref.generate(geom, n, 42, spheres)
        if reg is None:
            reg = ref.lib().ref_default_eta_reg(ref.domain_diameter(xyz), n)
        cfg = ref.make_config(leaf, tol=tol, cap=cap, kernel=kernel, structure=structure, reg=reg,
                              scale=scale)
        r = ref.RefRun(xyz, q, cfg).build()
        rec = structure_record(r)
        rec.update(dict(geometry=geom, n=n, leaf=leaf, tol=tol, cap=cap, kernel=kernel,
                        structure=structure, reg=reg, scale=scale, spheres=spheres,
                        points_fnv=fbits(xyz), near_fnv=fbits(r.leaf_dense())))
        try:
            r.factor()
        except RuntimeError as e:
            rec["factor_error"] = str(e)
            out["cases"][name] = rec
            print(name, "factor error", e)
            continue
        rec["ranks"] = {str(l): rk.tolist() for l, rk in r.factor_levels()}
        lvl, dims = r.cutoff()
        rec["cutoff"] = [int(lvl), dims.tolist()]
        b = ref.splitmix_signed(n, 7)
        x = r.solve(b)
        rec["x_fnv"] = fbits(x)
        y = r.dense_matvec(x)
        rec["residual"] = float(np.linalg.norm(y - b) / np.linalg.norm(b))
        rec["stats"] = {k: v for k, v in r.stats().items() if k.startswith("flops") or k == "kernel_evals"}
        if n <= 2048:
            arrays[name + "_x"] = x
        out["cases"][name] = rec
        print(name, rec["residual"])
    for name, geom, n, leaf, spheres in STRUCTURE_ONLY:
        xyz, q = ref.generate(geom, n, 42, spheres)
        r = ref.RefRun(xyz, q, ref.make_config(leaf)).build()
        rec = structure_record(r)
        rec.update(dict(geometry=geom, n=n, leaf=leaf, spheres=spheres, points_fnv=fbits(xyz)))
        out["cases"][name] = rec
        print(name, "structure", rec["perm_fnv"])
    # primitive kernels on seeded random inputs
    rng = np.random.default_rng(2024)
    prims = {}
    for m, k, nn in [(5, 3, 7), (70, 90, 130), (150, 300, 40)]:
        a = rng.standard_normal((m, k)); b = rng.standard_normal((k, nn)); c = rng.standard_normal((m, nn))
        arrays[f"gemm_{m}_{k}_{nn}_a"], arrays[f"gemm_{m}_{k}_{nn}_b"], arrays[f"gemm_{m}_{k}_{nn}_c"] = a, b, c
        prims[f"gemm_{m}_{k}_{nn}"] = [fbits(ref.gemm(a, b)), fbits(ref.gemm(a, b, -1.0, c=c)),
                                       fbits(ref.gemm(a.T.copy(), b, transa=True))]
    for n in [1, 7, 100, 170, 300]:
        a = rng.standard_normal((n, n)) + 0.1 * n * np.eye(n)
        lu, perm = ref.lu_factor(a)
        arrays[f"lu_{n}_a"] = a
        rec = [fbits(lu), ref.fnv64(perm)]
        for kind in ["solve", "lower", "upper", "transpose", "right", "upper_right"]:
            x = rng.standard_normal((n, 9)) if kind in ("solve", "lower", "upper", "transpose") else rng.standard_normal((9, n))
            arrays[f"lu_{n}_{kind}_x"] = x
            rec.append(fbits(ref.lu_solve(lu, perm, x, kind)))
        prims[f"lu_{n}"] = rec
    out["primitives"] = prims
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)


if __name__ == "__main__":
    main()
