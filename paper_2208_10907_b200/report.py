"""Reference-compatible reports, sweeps and file formats for the B200 path.

* ``run_report(cfg)`` -> the ``h2ulv-report/1`` document of
  ``RunReport::to_json`` (report.cpp:182-237), field for field, with the
  quantities defined as in ``Pipeline::report`` (report.cpp:113-180).
* ``sweep(cfg, axis, values)`` -> the ``h2ulv-sweep/1`` CSV and JSON of the
  CLI's ``sweep`` command (h2ulv_main.cpp:108-152) without CLI11.
* ``write_point_cloud`` / ``read_point_cloud`` (geometry.cpp:97-119) and
  ``write_vector`` / ``read_vector`` (solve.cpp:249-268): the same ``%.17g``
  ASCII formats and error messages, so files move between the two.

``solve_rel_error`` is the reference's (report.cpp:170-178): b = A 1 by the
dense matvec (h2g_matvec, bitwise equal to matvec_dense_oracle), x_ref the
dense LU solution of A x = b (lu_factor(A, 1e-15) + solve, dense_solve_oracle,
solve.cpp:241-247, run on the device with the bit-exact LU primitives), and
rel_error(x, x_ref) (linalg.cpp:618-630), for N <= oracle_guard.
"""
import json

import numpy as np

from .pipeline import Pipeline


def write_point_cloud(xyz, q, path):
    try:
        f = open(path, "w")
    except OSError:
        raise RuntimeError("write_point_cloud: cannot open " + path)
    with f:
        for p, c in zip(np.asarray(xyz, dtype=np.float64), np.asarray(q, dtype=np.float64)):
            f.write("%.17g %.17g %.17g %.17g\n" % (p[0], p[1], p[2], c))


def read_point_cloud(path):
    try:
        f = open(path)
    except OSError:
        raise RuntimeError("read_point_cloud: cannot open " + path)
    with f:
        vals = f.read().split()
    n = len(vals) // 4
    if n < 2:
        raise RuntimeError("read_point_cloud: fewer than 2 points")
    a = np.array(vals[: 4 * n], dtype=np.float64).reshape(n, 4)
    return np.ascontiguousarray(a[:, :3]), np.ascontiguousarray(a[:, 3])


def write_vector(v, path):
    try:
        f = open(path, "w")
    except OSError:
        raise RuntimeError("write_vector: cannot open " + path)
    with f:
        for x in np.asarray(v, dtype=np.float64).reshape(len(v), -1)[:, 0]:
            f.write("%.17g\n" % x)


def read_vector(path):
    try:
        f = open(path)
    except OSError:
        raise RuntimeError("read_vector: cannot open " + path)
    with f:
        return np.array(f.read().split(), dtype=np.float64)


def _config_json(cfg):
    c = {"n": cfg.n, "leaf_size": cfg.leaf_size, "tol": cfg.tol}
    if cfg.cap is not None:
        c["cap"] = cfg.cap
    c["kernel"] = cfg.kernel
    if cfg.kernel == "yukawa":
        c["alpha_m"] = cfg.alpha_m
    c["reg"] = cfg.reg if cfg.reg is not None else -1.0
    c["geometry"] = cfg.geometry
    if cfg.geometry == "sphere":
        c["spheres"] = cfg.spheres
        c["spacing"] = cfg.spacing
    c["admissibility"] = "weak" if cfg.structure in ("hss", "blr2") else "strong"
    c["eta"] = cfg.eta
    c["structure"] = cfg.structure
    c["variant"] = "nodep"
    c["threads"] = cfg.threads
    c["seed"] = cfg.seed
    return c


def run_report(cfg):
    """run_pipeline (report.cpp:239-243) -> h2ulv-report/1 as a dict."""
    pipe = Pipeline(cfg)
    try:
        return report_of(pipe)
    finally:
        if pipe.prob is not None:
            pipe.prob.close()


def report_of(pipe):
    """Pipeline::report (report.cpp:113-180) of a pipeline (factored on demand)."""
    cfg = pipe.cfg
    pipe.factor()
    p = pipe.prob
    st = p.stats()
    # the reference's phase keys (flops.cpp phase_name), in its std::map order
    flops = {"assemble": st["flops_assemble"], "fill_precompute": st["flops_fills"],
             "basis": st["flops_basis"], "skeleton": st["flops_skeleton"],
             "factorize": st["flops_factorize"], "solve": st["flops_solve"], "oracle": 0, "other": 0}
    walls = {k: 0.0 for k in flops}
    for k, v in p.phase_seconds().items():
        # driver sub-phases ("skeleton_leaf_pieces") fold into their reference phase
        base = next((ph for ph in flops if k == ph or k.startswith(ph + "_")), "other")
        walls[base] += v
    walls["assemble"] = st["t_tree"] + st["t_classify"] + st["t_near"]
    levels_n = p.levels
    flev = {lvl: ranks for lvl, ranks in p.factor_levels()}
    rep_levels = []
    for lvl in range(1, levels_n + 1):
        dense = int(p.L.h2g_list_count(p.h, lvl, 0))
        far = int(p.L.h2g_list_count(p.h, lvl, 1))
        ls = {"level": lvl, "dense_blocks": dense, "lowrank_blocks": far, "max_rank": 0, "mean_rank": 0.0}
        if lvl in flev:
            r = [int(x) for x in flev[lvl]]
            if r:
                ls["max_rank"] = max(r)
                ls["mean_rank"] = float(sum(r)) / len(r)
        rep_levels.append(ls)
    # factors_.levels.back() is the coarsest factorized level.
    top_level_max_rank = next((ls["max_rank"] for ls in rep_levels if ls["level"] == min(flev)), 0) if flev else 0
    max_leaf_rank = next((ls["max_rank"] for ls in rep_levels if ls["level"] == levels_n), 0) if flev else 0
    # Stored entries (report.cpp:149-157): leaf dense blocks, both bases of every
    # factorized box (dim^2 each), the elimination factors, the top LU.
    entries = int(p.L.h2g_near_entries(p.h))
    for lvl, ranks in flev.items():
        for k in range(len(ranks)):
            v = p.L.h2g_basis(p.h, lvl, k, 0, None)
            dim, rank = v & 0xFFFFFFFF, v >> 32
            entries += 2 * dim * dim
            rdim, sdim = dim - rank, rank
            entries += rdim * rdim + 2 * rdim * sdim
    top_n = int(p.L.h2g_top_n(p.h))
    entries += top_n * top_n
    rep = {
        "schema": "h2ulv-report/1",
        "config": _config_json(cfg),
        "wall_seconds": walls,
        "flops": flops,
        "total_flops": int(sum(flops.values())),
        "factorization_flops": int(flops["fill_precompute"] + flops["factorize"]),
        "kernel_evals": st["kernel_evals"],
        "total_seconds": pipe.build_seconds + pipe.factor_seconds,
        "levels": rep_levels,
        "top_level_max_rank": top_level_max_rank,
        "max_leaf_rank": max_leaf_rank,
        "dense_blocks_leaf": int(p.L.h2g_list_count(p.h, levels_n, 0)),
        "stored_entries": entries,
        "memory_bytes": entries * 8,
        "max_fill_residual_rel": p.max_fill_residual(),
        "dependency_edges": 0,  # nodep: no intra-level dependencies (ulv.cpp:1184-1193)
        "solve_rel_error": -1.0,
    }
    if cfg.oracle and cfg.n <= cfg.oracle_guard:
        rep["solve_rel_error"] = dense_oracle_error(pipe)
    return rep


def dense_oracle_error(pipe):
    """rel_error(x, x_ref) of Pipeline::report's oracle check (report.cpp:170-178)."""
    from . import _lib
    p = pipe.prob
    n = pipe.cfg.n
    b = p.matvec(np.ones(n))
    k = pipe.kernel
    A = _lib.assemble_block(k["kind"], k["alpha_m"], k["scale"], k["reg"], pipe.xyz, pipe.q, (0, n), (0, n))
    lu, perm = _lib.lu_factor(A, 1e-15)
    x_ref = _lib.lu_solve(lu, perm, b.reshape(n, 1), "solve")[:, 0]
    x = pipe.solve_rhs(b)
    den = float(np.sum(x_ref * x_ref))
    if den == 0.0:
        raise ValueError("rel_error: reference is zero")
    return float(np.sqrt(np.sum((x - x_ref) ** 2) / den))


def sweep(cfg, axis, values):
    """The CLI sweep command (h2ulv_main.cpp:108-152): (csv text, json dict)."""
    import copy
    csv = ("# h2ulv-sweep/1\naxis_value,factorize_seconds,total_flops,"
           "factorization_flops,max_rank,error,status\n")
    series = []
    for v in values:
        c = copy.copy(cfg)
        if axis == "n":
            c.n = int(v)
        elif axis == "leaf":
            c.leaf_size = int(v)
        elif axis == "tol":
            c.tol = float(v)
        elif axis == "threads":
            c.threads = int(v)
        else:
            raise RuntimeError("unknown sweep axis " + axis)
        try:
            rep = run_report(c)
            ftime = rep["wall_seconds"].get("fill_precompute", 0.0) + rep["wall_seconds"].get("factorize", 0.0)
            max_rank = max((l["max_rank"] for l in rep["levels"]), default=0)
            csv += "%g,%.6f,%d,%d,%d,%.3e,ok\n" % (v, ftime, rep["total_flops"], rep["factorization_flops"],
                                                  max_rank, rep["solve_rel_error"])
            rep["axis_value"] = v
            series.append(rep)
        except Exception as e:  # noqa: BLE001 — the CLI records the failure and continues
            csv += "%g,nan,0,0,0,nan,failed\n" % v
            series.append({"axis_value": v, "status": "failed: " + str(e)})
    return csv, {"schema": "h2ulv-sweep/1", "axis": axis, "series": series}


def report_json(cfg):
    """RunReport::to_json (two-space indent) of run_pipeline(cfg)."""
    return json.dumps(run_report(cfg), indent=2)
