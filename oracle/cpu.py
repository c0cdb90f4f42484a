"""TEST INFRASTRUCTURE ONLY: ctypes wrapper over oracle/liboracle.so, our C
restatement of the bit-exact front half (see h2oracle.c)."""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None
P = ctypes.c_void_p
i64 = ctypes.c_int64


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"C oracle not built: {LIB_PATH} (run make -C oracle liboracle.so)")
        L = ctypes.CDLL(LIB_PATH)
        L.or_generate.argtypes = [ctypes.c_int, i64, ctypes.c_uint64, i64, ctypes.c_double, P, P]
        L.or_domain_diameter.argtypes = [i64, P]
        L.or_domain_diameter.restype = ctypes.c_double
        L.or_default_eta_reg.argtypes = [ctypes.c_double, i64]
        L.or_default_eta_reg.restype = ctypes.c_double
        L.or_tree_levels.argtypes = [i64, i64]
        L.or_build_tree.argtypes = [i64, i64, P, P, P, P, P]
        L.or_classify.argtypes = [ctypes.c_int, P, ctypes.c_double, ctypes.c_int, P, P, P, P, P, P]
        L.or_assemble_block.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_double, P, P, i64, i64, i64, i64, P]
        L.or_fnv64.argtypes = [P, i64]
        L.or_fnv64.restype = ctypes.c_uint64
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


GEOMETRY = {"cube": 0, "line": 1, "sphere": 2}


def generate(geometry, n, seed, spheres=1, spacing=3.0):
    xyz = np.zeros((n, 3))
    q = np.zeros(n)
    if lib().or_generate(GEOMETRY[geometry], n, seed, spheres, spacing, _p(xyz), _p(q)):
        raise ValueError("or_generate failed")
    return xyz, q


def domain_diameter(xyz):
    xyz = np.ascontiguousarray(xyz, dtype=np.float64)
    return lib().or_domain_diameter(len(xyz), _p(xyz))


def default_eta_reg(diam, n):
    return lib().or_default_eta_reg(diam, n)


def build_tree(xyz, q, leaf):
    """Returns (xyz_reordered, q_reordered, order, nodes_be, nodes_geo, levels)."""
    xyz = np.array(xyz, dtype=np.float64, order="C")
    q = np.array(q, dtype=np.float64)
    n = len(q)
    L = lib().or_tree_levels(n, leaf)
    nn = (1 << (L + 1)) - 1
    order = np.zeros(n, dtype=np.int64)
    be = np.zeros((nn, 2), dtype=np.int64)
    geo = np.zeros((nn, 4))
    rc = lib().or_build_tree(n, leaf, _p(xyz), _p(q), _p(order), _p(be), _p(geo))
    if rc:
        raise ValueError(f"or_build_tree failed ({rc})")
    return xyz, q, order, be, geo, L


def classify(levels, geo, eta=1.0, weak=False):
    """Per-level CSR lists: {lvl: (near_ptr, near_idx, far_ptr, far_idx)}."""
    geo = np.ascontiguousarray(geo, dtype=np.float64)
    nt = np.zeros(1, dtype=np.int64)
    ft = np.zeros(1, dtype=np.int64)
    lib().or_classify(levels, _p(geo), eta, int(weak), None, None, None, None, _p(nt), _p(ft))
    rows = (1 << (levels + 1)) - 2
    nptr = np.zeros(rows + 1, dtype=np.int64)
    fptr = np.zeros(rows + 1, dtype=np.int64)
    nidx = np.zeros(max(int(nt[0]), 1), dtype=np.int64)
    fidx = np.zeros(max(int(ft[0]), 1), dtype=np.int64)
    lib().or_classify(levels, _p(geo), eta, int(weak), _p(nptr), _p(nidx), _p(fptr), _p(fidx),
                      _p(nt), _p(ft))
    out = {}
    for lvl in range(1, levels + 1):
        g0 = (1 << lvl) - 2
        m = 1 << lvl
        npt = nptr[g0:g0 + m + 1]
        fpt = fptr[g0:g0 + m + 1]
        out[lvl] = (npt - npt[0], nidx[npt[0]:npt[-1]].copy(), fpt - fpt[0],
                    fidx[fpt[0]:fpt[-1]].copy())
    return out


def assemble_block(xyz, q, rows, cols, kind="laplace", alpha_m=0.0, scale=4 * np.pi, reg=0.0):
    xyz = np.ascontiguousarray(xyz, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    out = np.zeros((rows[1] - rows[0], cols[1] - cols[0]), order="F")
    rc = lib().or_assemble_block({"laplace": 0, "yukawa": 1, "gaussian": 2}[kind], alpha_m, scale, reg, _p(xyz),
                                 _p(q), rows[0], rows[1], cols[0], cols[1], _p(out))
    if rc:
        raise RuntimeError("assemble_block: singular evaluation (r + eta_reg == 0)")
    return out


def fnv64(values):
    v = np.ascontiguousarray(values, dtype=np.int64)
    return int(lib().or_fnv64(_p(v), len(v)))
