"""TEST INFRASTRUCTURE ONLY: ctypes wrapper over oracle/_ref/libh2ref.so.

libh2ref.so is the unmodified reference (proj/src/*.cpp) plus
oracle/ref_shim.cpp, built by oracle/Makefile. See ref_shim.cpp for the
reference entry points each function drives.
"""
import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# H2REF_LIB selects another build of the same sources (e.g. oracle/_ref_native,
# the reference's own -march=native flags; oracle/Makefile ref-native).
LIB_PATH = os.environ.get("H2REF_LIB") or os.path.join(_HERE, "_ref", "libh2ref.so")
# The reference with its covered-coupling defect corrected (oracle/fix_reference.py).
FIXED_PATH = os.path.join(_HERE, "_ref_fixed", "libh2ref.so")
_libs = {}

i64 = ctypes.c_int64
f64 = ctypes.c_double
P = ctypes.c_void_p


class RefConfig(ctypes.Structure):
    _fields_ = [
        ("leaf_size", i64), ("tol", f64), ("cap", i64), ("kernel", ctypes.c_int32),
        ("structure", ctypes.c_int32), ("alpha_m", f64), ("reg", f64), ("scale", f64),
        ("eta", f64), ("threads", ctypes.c_int32), ("absorb_coupling", ctypes.c_int32),
    ]


def available(path=None):
    return os.path.exists(path or LIB_PATH)


def fixed_available():
    return os.path.exists(FIXED_PATH)


def lib(path=None):
    path = path or LIB_PATH
    if path not in _libs:
        if not available(path):
            raise RuntimeError(f"reference oracle not built: {path} (run make -C oracle ref ref-fixed)")
        L = ctypes.CDLL(path)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_new.restype = P
        L.ref_new.argtypes = [i64, P, P]
        L.ref_free.argtypes = [P]
        for name in ("ref_build", "ref_factor"):
            getattr(L, name).argtypes = [P, ctypes.POINTER(RefConfig)]
        L.ref_levels.argtypes = [P]
        L.ref_tree_perm.argtypes = [P, P]
        L.ref_nodes.argtypes = [P, P, P]
        L.ref_reordered_points.argtypes = [P, P, P]
        L.ref_list_count.argtypes = [P, ctypes.c_int, ctypes.c_int]
        L.ref_list_count.restype = i64
        L.ref_list.argtypes = [P, ctypes.c_int, ctypes.c_int, P, P]
        L.ref_leaf_dense_entries.argtypes = [P]
        L.ref_leaf_dense_entries.restype = i64
        L.ref_leaf_dense.argtypes = [P, P]
        L.ref_stats.argtypes = [P, P, P]
        L.ref_num_factor_levels.argtypes = [P]
        L.ref_factor_level.argtypes = [P, ctypes.c_int, P]
        L.ref_cutoff.argtypes = [P, P]
        L.ref_cutoff.restype = i64
        L.ref_top_n.argtypes = [P]
        L.ref_top_n.restype = i64
        L.ref_top.argtypes = [P, P, P]
        L.ref_basis.argtypes = [P, ctypes.c_int, i64, ctypes.c_int, P]
        L.ref_basis.restype = i64
        L.ref_max_fill_residual.argtypes = [P]
        L.ref_max_fill_residual.restype = f64
        L.ref_solve.argtypes = [P, i64, P, P]
        L.ref_dense_matvec.argtypes = [P, P, P]
        L.ref_dense_solve.argtypes = [P, P, P]
        L.ref_generate.argtypes = [ctypes.c_int32, i64, ctypes.c_uint64, i64, f64, P, P]
        L.ref_domain_diameter.argtypes = [i64, P]
        L.ref_domain_diameter.restype = f64
        L.ref_default_eta_reg.argtypes = [f64, i64]
        L.ref_default_eta_reg.restype = f64
        L.ref_lu_factor.argtypes = [i64, P, f64, P, P]
        L.ref_basis_from_members.argtypes = [i64, i64, P, i64, P, f64, i64, i64, P, P]
        L.ref_gemm.argtypes = [i64, i64, i64, f64, P, ctypes.c_int, P, ctypes.c_int, ctypes.c_int, P]
        L.ref_lu_solve.argtypes = [i64, P, P, ctypes.c_int, i64, i64, P]
        _libs[path] = L
    return _libs[path]


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(rc, L=None):
    if rc != 0:
        raise RuntimeError((L or lib()).ref_last_error().decode())


GEOMETRY = {"cube": 0, "line": 1, "sphere": 2}


def generate(geometry, n, seed, spheres=1, spacing=3.0):
    xyz = np.zeros((n, 3))
    q = np.zeros(n)
    _check(lib().ref_generate(GEOMETRY[geometry], n, seed, spheres, spacing, _p(xyz), _p(q)))
    return xyz, q


def domain_diameter(xyz):
    xyz = np.ascontiguousarray(xyz, dtype=np.float64)
    return lib().ref_domain_diameter(len(xyz), _p(xyz))


def make_config(leaf_size, tol=1e-8, cap=None, kernel="laplace", structure="h2", alpha_m=1.0,
                reg=1e-3, scale=1.0, eta=1.0, threads=None, absorb_coupling=True):
    return RefConfig(leaf_size, tol, cap or 0, 0 if kernel == "laplace" else 1,
                     {"h2": 0, "hss": 1, "blr2": 2}[structure], alpha_m, reg, scale, eta,
                     threads or os.cpu_count(), 1 if absorb_coupling else 0)


class RefRun:
    """One reference pipeline over a given point cloud (original order)."""

    def __init__(self, xyz, q, cfg, fixed=False):
        """fixed=True: the corrected build (oracle/_ref_fixed, fix_reference.py)."""
        self.L = lib(FIXED_PATH if fixed else None)
        self.xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        self.q = np.ascontiguousarray(q, dtype=np.float64)
        self.n = len(self.q)
        self.cfg = cfg
        self.h = self.L.ref_new(self.n, _p(self.xyz), _p(self.q))

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_free(self.h)
            self.h = None

    def build(self):
        _check(self.L.ref_build(self.h, ctypes.byref(self.cfg)), self.L)
        return self

    def factor(self):
        _check(self.L.ref_factor(self.h, ctypes.byref(self.cfg)), self.L)
        return self

    @property
    def levels(self):
        return self.L.ref_levels(self.h)

    def perm(self):
        out = np.zeros(self.n, dtype=np.int64)
        self.L.ref_tree_perm(self.h, _p(out))
        return out

    def nodes(self):
        nn = (1 << (self.levels + 1)) - 1
        be = np.zeros((nn, 2), dtype=np.int64)
        geo = np.zeros((nn, 4))
        self.L.ref_nodes(self.h, _p(be), _p(geo))
        return be, geo

    def reordered(self):
        xyz = np.zeros((self.n, 3))
        q = np.zeros(self.n)
        self.L.ref_reordered_points(self.h, _p(xyz), _p(q))
        return xyz, q

    def lists(self, lvl, far):
        cnt = self.L.ref_list_count(self.h, lvl, 1 if far else 0)
        ptr = np.zeros((1 << lvl) + 1, dtype=np.int64)
        idx = np.zeros(max(cnt, 1), dtype=np.int64)
        self.L.ref_list(self.h, lvl, 1 if far else 0, _p(ptr), _p(idx))
        return ptr, idx[:cnt]

    def leaf_dense(self):
        out = np.zeros(self.L.ref_leaf_dense_entries(self.h))
        self.L.ref_leaf_dense(self.h, _p(out))
        return out

    def stats(self):
        t = np.zeros(5)
        f = np.zeros(6, dtype=np.uint64)
        self.L.ref_stats(self.h, _p(t), _p(f))
        return dict(t_tree=t[0], t_classify=t[1], t_near=t[2], t_factor=t[3], t_solve=t[4],
                    flops_fills=int(f[0]), flops_basis=int(f[1]), flops_skeleton=int(f[2]),
                    flops_factorize=int(f[3]), kernel_evals=int(f[4]), metric_flops=int(f[5]))

    def factor_levels(self):
        out = []
        for li in range(self.L.ref_num_factor_levels(self.h)):
            ranks = np.zeros(1 << self.levels, dtype=np.int64)
            lvl = self.L.ref_factor_level(self.h, li, _p(ranks))
            out.append((lvl, ranks[: 1 << lvl].copy()))
        return out

    def cutoff(self):
        dims = np.zeros(1 << self.levels, dtype=np.int64)
        v = self.L.ref_cutoff(self.h, _p(dims))
        m = v & 0xFFFFFFFF
        return v >> 32, dims[:m].copy()

    def top(self):
        n = self.L.ref_top_n(self.h)
        lu = np.zeros((n, n), order="F")
        perm = np.zeros(n, dtype=np.int64)
        self.L.ref_top(self.h, _p(lu), _p(perm))
        return lu, perm

    def basis(self, lvl, k, side):
        v = self.L.ref_basis(self.h, lvl, k, side, None)
        dim, rank = v & 0xFFFFFFFF, v >> 32
        out = np.zeros((dim, dim), order="F")
        if dim:
            self.L.ref_basis(self.h, lvl, k, side, _p(out))
        return out, rank

    def max_fill_residual(self):
        return self.L.ref_max_fill_residual(self.h)

    def solve(self, b):
        b = np.asfortranarray(b, dtype=np.float64)
        nrhs = 1 if b.ndim == 1 else b.shape[1]
        x = np.zeros_like(b)
        _check(self.L.ref_solve(self.h, nrhs, _p(b), _p(x)), self.L)
        return x

    def dense_matvec(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.n)
        _check(self.L.ref_dense_matvec(self.h, _p(x), _p(y)), self.L)
        return y

    def dense_solve(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(self.n)
        _check(self.L.ref_dense_solve(self.h, _p(b), _p(x)), self.L)
        return x


def lu_factor(a, tol=1e-14):
    a = np.asfortranarray(a, dtype=np.float64)
    n = a.shape[0]
    lu = np.zeros((n, n), order="F")
    perm = np.zeros(n, dtype=np.int64)
    _check(lib().ref_lu_factor(n, _p(a), tol, _p(lu), _p(perm)))
    return lu, perm


def gemm(a, b, alpha=1.0, transa=False, transb=False, c=None):
    a = np.asfortranarray(a, dtype=np.float64)
    b = np.asfortranarray(b, dtype=np.float64)
    m = a.shape[1] if transa else a.shape[0]
    k = a.shape[0] if transa else a.shape[1]
    n = b.shape[0] if transb else b.shape[1]
    acc = c is not None
    out = np.array(c, dtype=np.float64, order="F") if acc else np.zeros((m, n), order="F")
    _check(lib().ref_gemm(m, n, k, alpha, _p(a), int(transa), _p(b), int(transb), int(acc), _p(out)))
    return out


def lu_solve(lu, perm, x, kind):
    lu = np.asfortranarray(lu, dtype=np.float64)
    perm = np.ascontiguousarray(perm, dtype=np.int64)
    x = np.array(x, dtype=np.float64, order="F")
    kinds = {"solve": 0, "lower": 1, "upper": 2, "transpose": 3, "right": 4, "upper_right": 5}
    _check(lib().ref_lu_solve(lu.shape[0], _p(lu), _p(perm), kinds[kind], x.shape[0], x.shape[1],
                              _p(x)))
    return x


def basis_from_members(concat, offsets, tol, cap=None, min_rank=0):
    concat = np.asfortranarray(concat, dtype=np.float64)
    dim = concat.shape[0]
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    q = np.zeros((dim, dim), order="F")
    rank = np.zeros(1, dtype=np.int64)
    _check(lib().ref_basis_from_members(dim, concat.shape[1], _p(concat), len(offsets) - 1,
                                        _p(offsets), tol, cap or 0, min_rank, _p(q), _p(rank)))
    return q, int(rank[0])


def fnv64(values):
    """FNV-1a over int64 values (h ^= (u64)v; h *= prime)."""
    h = 0xcbf29ce484222325
    for v in np.asarray(values, dtype=np.int64).view(np.uint64).tolist():
        h ^= v
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def splitmix_signed(n, seed):
    """b_i = SplitMix64(seed).next_signed() (prng.hpp:14-25), vectorised."""
    k = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + k * np.uint64(0x9e3779b97f4a7c15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94d049bb133111eb)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return 2.0 * u - 1.0
