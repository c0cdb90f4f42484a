"""ctypes binding of include/h2g.h (libh2g.so, built in-tree by `make`)."""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(_HERE, "libh2g.so")
_lib = None

i64 = ctypes.c_int64
f64 = ctypes.c_double
P = ctypes.c_void_p


class H2GError(RuntimeError):
    """Raised with the reference's error message (h2g_last_error)."""


class Kernel(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("alpha_m", f64), ("permittivity_scale", f64),
                ("eta_reg", f64)]


class Options(ctypes.Structure):
    _fields_ = [("tol", f64), ("cap", i64), ("rr_pivot_tol", f64), ("absorb_coupling", ctypes.c_int32),
                ("abort_residual_factor", f64), ("structure", ctypes.c_int32), ("eta", f64),
                ("qr_mem_budget", i64), ("qr_mode", ctypes.c_int32),
                ("reference_compat", ctypes.c_int32)]


EXPORTS = [
    "h2g_last_error", "h2g_version", "h2g_create", "h2g_destroy", "h2g_set_kernel",
    "h2g_set_options", "h2g_build", "h2g_build_dev", "h2g_factor", "h2g_solve", "h2g_solve_dev",
    "h2g_levels", "h2g_tree_perm", "h2g_nodes", "h2g_reordered_points", "h2g_list_count",
    "h2g_list", "h2g_near_entries", "h2g_near_dense", "h2g_num_factor_levels",
    "h2g_factor_level", "h2g_cutoff", "h2g_top_n", "h2g_top", "h2g_basis",
    "h2g_max_fill_residual", "h2g_stats", "h2g_matvec", "h2g_lu_factor",
    "h2g_basis_from_members", "h2g_basis_from_members_mode", "h2g_lu_solve", "h2g_gemm", "h2g_stats_dev", "h2g_set_profile",
    "h2g_reset_profile", "h2g_kernel_stats", "h2g_set_stream", "h2g_phase_seconds",
    "h2g_nccl_unique_id", "h2g_comm_nccl", "h2g_comm_host", "h2g_comm_destroy", "h2g_set_comm",
    "h2g_partition_range", "h2g_kernel_evals", "h2g_generate_points", "h2g_points_last_error",
    "h2g_exp_glibc_host", "h2g_level_dims", "h2g_level_block", "h2g_level_lu", "h2g_level_elim",
    "h2g_assemble_block", "h2g_set_sampling", "h2g_trim_memory",
]

# h2g_host_allgather_fn (include/h2g.h)
HostAllgatherFn = ctypes.CFUNCTYPE(ctypes.c_int, P, P, ctypes.POINTER(i64), ctypes.c_int)


def lib():
    """Load libh2g.so; raise loudly if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(lib_path):
            raise H2GError(f"libh2g.so not built at {lib_path}; run `make -C paper_2208_10907_b200`")
        L = ctypes.CDLL(lib_path)
        L.h2g_last_error.restype = ctypes.c_char_p
        L.h2g_points_last_error.restype = ctypes.c_char_p
        L.h2g_exp_glibc_host.argtypes = [i64, P, P]
        L.h2g_level_dims.argtypes = [P, ctypes.c_int, P, P, P]
        L.h2g_level_block.argtypes = [P, ctypes.c_int, i64, i64, P, P, P]
        L.h2g_assemble_block.argtypes = [ctypes.POINTER(Kernel), i64, P, P, i64, i64, i64, i64, P]
        L.h2g_generate_points.argtypes = [ctypes.c_int32, i64, ctypes.c_uint64, i64, f64, P, P]
        L.h2g_create.argtypes = [ctypes.POINTER(P)]
        L.h2g_destroy.argtypes = [P]
        L.h2g_set_kernel.argtypes = [P, ctypes.POINTER(Kernel)]
        L.h2g_set_options.argtypes = [P, ctypes.POINTER(Options)]
        L.h2g_set_sampling.argtypes = [P, i64]
        L.h2g_trim_memory.argtypes = []
        L.h2g_trim_memory.restype = None
        L.h2g_build.argtypes = [P, i64, P, P, i64]
        L.h2g_build_dev.argtypes = [P, i64, P, P, i64]
        L.h2g_factor.argtypes = [P]
        L.h2g_solve.argtypes = [P, i64, P, P]
        L.h2g_solve_dev.argtypes = [P, i64, P, P]
        L.h2g_levels.argtypes = [P]
        L.h2g_tree_perm.argtypes = [P, P]
        L.h2g_nodes.argtypes = [P, P, P]
        L.h2g_reordered_points.argtypes = [P, P, P]
        L.h2g_list_count.argtypes = [P, ctypes.c_int, ctypes.c_int]
        L.h2g_list_count.restype = i64
        L.h2g_list.argtypes = [P, ctypes.c_int, ctypes.c_int, P, P]
        L.h2g_near_entries.argtypes = [P]
        L.h2g_near_entries.restype = i64
        L.h2g_near_dense.argtypes = [P, P]
        L.h2g_num_factor_levels.argtypes = [P]
        L.h2g_factor_level.argtypes = [P, ctypes.c_int, P]
        L.h2g_cutoff.argtypes = [P, P]
        L.h2g_cutoff.restype = i64
        L.h2g_top_n.argtypes = [P]
        L.h2g_top_n.restype = i64
        L.h2g_top.argtypes = [P, P, P]
        L.h2g_basis.argtypes = [P, ctypes.c_int, i64, ctypes.c_int, P]
        L.h2g_basis.restype = i64
        L.h2g_max_fill_residual.argtypes = [P]
        L.h2g_max_fill_residual.restype = f64
        L.h2g_stats.argtypes = [P, P, P, P]
        L.h2g_matvec.argtypes = [P, i64, P, P]
        L.h2g_lu_factor.argtypes = [i64, P, f64, P, P]
        L.h2g_basis_from_members.argtypes = [i64, i64, P, i64, P, f64, i64, i64, P, P]
        L.h2g_basis_from_members_mode.argtypes = [i64, i64, P, i64, P, f64, i64, i64, ctypes.c_int32, P, P]
        L.h2g_lu_solve.argtypes = [i64, P, P, ctypes.c_int, i64, i64, P]
        L.h2g_gemm.argtypes = [i64, i64, i64, f64, P, ctypes.c_int, P, ctypes.c_int, ctypes.c_int, P]
        L.h2g_stats_dev.argtypes = [P, P]
        L.h2g_set_stream.argtypes = [P, P]
        L.h2g_phase_seconds.argtypes = [P, ctypes.c_int, ctypes.c_char_p, ctypes.c_int, P]
        L.h2g_set_profile.argtypes = [P, ctypes.c_int]
        L.h2g_reset_profile.argtypes = [P]
        L.h2g_kernel_stats.argtypes = [P, ctypes.c_int, ctypes.c_char_p, ctypes.c_int, P, P, P, P]
        L.h2g_nccl_unique_id.argtypes = [P]
        L.h2g_comm_nccl.argtypes = [ctypes.c_int, ctypes.c_int, P, ctypes.POINTER(P)]
        L.h2g_comm_host.argtypes = [ctypes.c_int, ctypes.c_int, HostAllgatherFn, P, ctypes.POINTER(P)]
        L.h2g_comm_destroy.argtypes = [P]
        L.h2g_set_comm.argtypes = [P, P]
        L.h2g_partition_range.argtypes = [i64, ctypes.c_int, ctypes.c_int, P, P]
        L.h2g_kernel_evals.argtypes = [P]
        L.h2g_kernel_evals.restype = i64
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def partition_range(m, nranks, rank):
    """Boxes [lo, hi) of an m-box level owned by rank (h2g_partition_range)."""
    lo, hi = i64(), i64()
    _check(lib().h2g_partition_range(m, nranks, rank, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def nccl_unique_id():
    """128-byte ncclUniqueId (create on rank 0, broadcast to the others)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().h2g_nccl_unique_id(buf))
    return buf.raw


class Comm:
    """h2g_comm: the multi-GPU level partition's communicator (one per rank,
    shared by any number of problems)."""

    def __init__(self, h, cb=None):
        self.h, self._cb = h, cb

    @classmethod
    def nccl(cls, nranks, rank, unique_id):
        h = P()
        _check(lib().h2g_comm_nccl(nranks, rank, ctypes.c_char_p(unique_id), ctypes.byref(h)))
        return cls(h)

    @classmethod
    def host(cls, nranks, rank, fn):
        cb = HostAllgatherFn(fn)
        h = P()
        _check(lib().h2g_comm_host(nranks, rank, cb, None, ctypes.byref(h)))
        return cls(h, cb)

    def close(self):
        if self.h:
            lib().h2g_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gloo_allgather(group=None):
    """A host all-gather-v callback over a torch.distributed (gloo) group, for
    h2g_set_comm_host: the segments are padded to the longest and gathered."""
    import torch
    import torch.distributed as dist

    def fn(user, host_buf, offs, nranks):
        try:
            o = [offs[r] for r in range(nranks + 1)]
            sizes = [o[r + 1] - o[r] for r in range(nranks)]
            me = dist.get_rank(group)
            buf = (ctypes.c_uint8 * o[nranks]).from_address(host_buf)
            arr = np.ctypeslib.as_array(buf)
            mx = max(max(sizes), 1)
            mine = torch.zeros(mx, dtype=torch.uint8)
            mine[:sizes[me]] = torch.from_numpy(arr[o[me]:o[me + 1]].copy())
            got = [torch.empty(mx, dtype=torch.uint8) for _ in range(nranks)]
            dist.all_gather(got, mine, group=group)
            for r in range(nranks):
                if r != me and sizes[r]:
                    arr[o[r]:o[r + 1]] = got[r][:sizes[r]].numpy()
            return 0
        except Exception:  # reported as a failed exchange by the library
            import traceback
            traceback.print_exc()
            return 1
    return fn


def _check(rc):
    if rc != 0:
        raise H2GError(lib().h2g_last_error().decode())


class Problem:
    """One device-resident H2 problem: tree, structure, near field, factors."""

    def __init__(self):
        L = lib()
        h = P()
        _check(L.h2g_create(ctypes.byref(h)))
        self.L = L
        self.h = h
        self.n = 0

    def close(self):
        if getattr(self, "h", None):
            self.L.h2g_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def set_kernel(self, kind="laplace", alpha_m=0.0, scale=4 * np.pi, reg=0.0):
        k = Kernel({"laplace": 0, "yukawa": 1, "gaussian": 2}[kind], alpha_m, scale, reg)
        _check(self.L.h2g_set_kernel(self.h, ctypes.byref(k)))

    def set_options(self, tol=1e-8, cap=None, rr_pivot_tol=1e-13, absorb_coupling=True,
                    abort_residual_factor=100.0, structure="h2", eta=1.0, qr_mem_budget=0, qr_mode="exact",
                    reference_compat=True, sample_cols=0):
        o = Options(tol, cap or 0, rr_pivot_tol, 1 if absorb_coupling else 0, abort_residual_factor,
                    {"h2": 0, "hss": 1, "blr2": 2}[structure], eta, qr_mem_budget, {"exact": 0, "blocked": 1, "compressed": 2}[qr_mode],
                    1 if reference_compat else 0)
        _check(self.L.h2g_set_options(self.h, ctypes.byref(o)))
        # B200 extension: strided sampling of wide far-field basis members (0 = the reference's members).
        _check(self.L.h2g_set_sampling(self.h, int(sample_cols or 0)))

    def build(self, xyz, q, leaf):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        q = np.ascontiguousarray(q, dtype=np.float64)
        self.n = len(q)
        _check(self.L.h2g_build(self.h, self.n, _p(xyz), _p(q), leaf))

    def build_dev(self, xyz_ptr, q_ptr, n, leaf):
        self.n = n
        _check(self.L.h2g_build_dev(self.h, n, xyz_ptr, q_ptr, leaf))

    def factor(self):
        _check(self.L.h2g_factor(self.h))

    def solve(self, b):
        b = np.asfortranarray(b, dtype=np.float64)
        nrhs = 1 if b.ndim == 1 else b.shape[1]
        x = np.zeros_like(b)
        _check(self.L.h2g_solve(self.h, nrhs, _p(b), _p(x)))
        return x

    def solve_dev(self, b_ptr, x_ptr, nrhs=1):
        _check(self.L.h2g_solve_dev(self.h, nrhs, b_ptr, x_ptr))

    def matvec(self, x):
        x = np.asfortranarray(x, dtype=np.float64)
        nrhs = 1 if x.ndim == 1 else x.shape[1]
        y = np.zeros_like(x)
        _check(self.L.h2g_matvec(self.h, nrhs, _p(x), _p(y)))
        return y

    # ---- inspection ----
    @property
    def levels(self):
        return self.L.h2g_levels(self.h)

    def perm(self):
        out = np.zeros(self.n, dtype=np.int64)
        _check(self.L.h2g_tree_perm(self.h, _p(out)))
        return out

    def nodes(self):
        nn = (1 << (self.levels + 1)) - 1
        be = np.zeros((nn, 2), dtype=np.int64)
        geo = np.zeros((nn, 4))
        _check(self.L.h2g_nodes(self.h, _p(be), _p(geo)))
        return be, geo

    def reordered(self):
        xyz = np.zeros((self.n, 3))
        q = np.zeros(self.n)
        _check(self.L.h2g_reordered_points(self.h, _p(xyz), _p(q)))
        return xyz, q

    def lists(self, lvl, far):
        cnt = self.L.h2g_list_count(self.h, lvl, 1 if far else 0)
        if cnt < 0:
            raise RuntimeError(self.L.h2g_last_error().decode())
        ptr = np.zeros((1 << lvl) + 1, dtype=np.int64)
        idx = np.zeros(max(cnt, 1), dtype=np.int64)
        _check(self.L.h2g_list(self.h, lvl, 1 if far else 0, _p(ptr), _p(idx)))
        return ptr, idx[:cnt]

    def leaf_dense(self):
        out = np.zeros(self.L.h2g_near_entries(self.h))
        _check(self.L.h2g_near_dense(self.h, _p(out)))
        return out

    def factor_levels(self):
        out = []
        for li in range(self.L.h2g_num_factor_levels(self.h)):
            ranks = np.zeros(1 << self.levels, dtype=np.int64)
            lvl = self.L.h2g_factor_level(self.h, li, _p(ranks))
            if lvl < 0:
                raise RuntimeError(self.L.h2g_last_error().decode())
            out.append((lvl, ranks[: 1 << lvl].copy()))
        return out

    def cutoff(self):
        dims = np.zeros(1 << self.levels, dtype=np.int64)
        v = self.L.h2g_cutoff(self.h, _p(dims))
        return v >> 32, dims[: v & 0xFFFFFFFF].copy()

    def top(self):
        n = self.L.h2g_top_n(self.h)
        lu = np.zeros((n, n), order="F")
        perm = np.zeros(n, dtype=np.int64)
        _check(self.L.h2g_top(self.h, _p(lu), _p(perm)))
        return lu, perm

    def basis(self, lvl, k, side):
        v = self.L.h2g_basis(self.h, lvl, k, side, None)
        if v < 0:
            raise RuntimeError(self.L.h2g_last_error().decode())
        dim, rank = v & 0xFFFFFFFF, v >> 32
        out = np.zeros((dim, dim), order="F")
        if dim:
            self.L.h2g_basis(self.h, lvl, k, side, _p(out))
        return out, rank

    def level_block(self, li, i, j):
        """DenseSystem::block(i, j) of factorized level li (h2g_level_block)."""
        r, c = ctypes.c_int64(), ctypes.c_int64()
        _check(self.L.h2g_level_block(self.h, li, i, j, ctypes.byref(r), ctypes.byref(c), None))
        out = np.zeros((r.value, c.value), order="F")
        if out.size:
            _check(self.L.h2g_level_block(self.h, li, i, j, ctypes.byref(r), ctypes.byref(c), _p(out)))
        return out

    def level_dims(self, li):
        m = self.L.h2g_level_dims(self.h, li, None, None, None)
        if m < 0:
            raise H2GError(self.L.h2g_last_error().decode())
        dims = np.zeros(m, dtype=np.int64)
        ranks = np.zeros(m, dtype=np.int64)
        z = ctypes.c_int32()
        self.L.h2g_level_dims(self.h, li, _p(dims), _p(ranks), ctypes.byref(z))
        return dims, ranks, bool(z.value)

    def set_stream(self, stream_ptr):
        _check(self.L.h2g_set_stream(self.h, stream_ptr))

    def set_comm(self, comm):
        """Partition the factorization over comm's ranks (None: single GPU)."""
        self._comm = comm  # the callback (if any) stays alive with the problem
        _check(self.L.h2g_set_comm(self.h, comm.h if comm is not None else None))

    def stats_dev(self):
        t = np.zeros(3)
        self.L.h2g_stats_dev(self.h, _p(t))
        return dict(build=t[0], factor=t[1], solve=t[2])

    def set_profile(self, on=True):
        self.L.h2g_set_profile(self.h, 1 if on else 0)

    def reset_profile(self):
        self.L.h2g_reset_profile(self.h)

    def kernel_stats(self):
        out = {}
        idx = 0
        while True:
            name = ctypes.create_string_buffer(64)
            ms, fl, by = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
            n = ctypes.c_int64()
            if not self.L.h2g_kernel_stats(self.h, idx, name, 64, ctypes.byref(ms), ctypes.byref(n),
                                           ctypes.byref(fl), ctypes.byref(by)):
                break
            out[name.value.decode()] = dict(ms=ms.value, launches=n.value, flops=fl.value, bytes=by.value)
            idx += 1
        return out

    def phase_seconds(self):
        out = {}
        idx = 0
        while True:
            name = ctypes.create_string_buffer(64)
            sec = ctypes.c_double()
            if not self.L.h2g_phase_seconds(self.h, idx, name, 64, ctypes.byref(sec)):
                break
            out[name.value.decode()] = sec.value
            idx += 1
        return out

    def max_fill_residual(self):
        return self.L.h2g_max_fill_residual(self.h)

    def stats(self):
        t = np.zeros(5)
        f = np.zeros(6)
        n = ctypes.c_int64(0)
        self.L.h2g_stats(self.h, _p(t), _p(f), ctypes.byref(n))
        return dict(t_tree=t[0], t_classify=t[1], t_near=t[2], t_factor=t[3], t_solve=t[4],
                    kernel_evals=int(self.L.h2g_kernel_evals(self.h)),
                    flops_fills=f[0], flops_basis=f[1], flops_skeleton=f[2], flops_factorize=f[3],
                    flops_assemble=f[4], flops_solve=f[5], launches=n.value)


# ---- single primitives ---------------------------------------------------
def lu_factor(a, tol=1e-14):
    a = np.asfortranarray(a, dtype=np.float64)
    n = a.shape[0]
    lu = np.zeros((n, n), order="F")
    perm = np.zeros(n, dtype=np.int64)
    _check(lib().h2g_lu_factor(n, _p(a), tol, _p(lu), _p(perm)))
    return lu, perm


def lu_solve(lu, perm, x, kind):
    lu = np.asfortranarray(lu, dtype=np.float64)
    perm = np.ascontiguousarray(perm, dtype=np.int64)
    x = np.array(x, dtype=np.float64, order="F")
    kinds = {"solve": 0, "lower": 1, "upper": 2, "transpose": 3, "right": 4, "upper_right": 5}
    _check(lib().h2g_lu_solve(lu.shape[0], _p(lu), _p(perm), kinds[kind], x.shape[0], x.shape[1],
                              _p(x)))
    return x


def gemm(a, b, alpha=1.0, transa=False, transb=False, c=None):
    a = np.asfortranarray(a, dtype=np.float64)
    b = np.asfortranarray(b, dtype=np.float64)
    m = a.shape[1] if transa else a.shape[0]
    k = a.shape[0] if transa else a.shape[1]
    n = b.shape[0] if transb else b.shape[1]
    acc = c is not None
    out = np.array(c, dtype=np.float64, order="F") if acc else np.zeros((m, n), order="F")
    _check(lib().h2g_gemm(m, n, k, alpha, _p(a), int(transa), _p(b), int(transb), int(acc), _p(out)))
    return out


def trim_memory():
    """h2g_trim_memory: return the arena's entirely free segments to the driver."""
    lib().h2g_trim_memory()


GEOMETRIES = {"cube": 0, "line": 1, "sphere": 2, "uniform_sphere": 3, "ellipsoids": 4}


def generate_points(geometry, n, seed, spheres=1, spacing=3.0):
    """h2g_generate_points: the reference's seeded generators bit for bit
    (geometry.cpp:42-95) plus uniform_sphere / ellipsoids (host code)."""
    L = lib()
    xyz = np.zeros((n, 3))
    q = np.zeros(n)
    if L.h2g_generate_points(GEOMETRIES[geometry], n, seed, spheres, spacing, _p(xyz), _p(q)) != 0:
        raise H2GError(L.h2g_points_last_error().decode())
    return xyz, q


def assemble_block(kind, alpha_m, scale, reg, xyz, q, rows, cols):
    """assemble_block (kernels.cpp:242-268) of a host cloud, evaluated on the
    device (h2g_assemble_block): rows/cols are (begin, end) index ranges."""
    xyz = np.ascontiguousarray(xyz, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    k = Kernel({"laplace": 0, "yukawa": 1, "gaussian": 2}[kind], alpha_m, scale, reg)
    out = np.zeros((rows[1] - rows[0], cols[1] - cols[0]), order="F")
    _check(lib().h2g_assemble_block(ctypes.byref(k), len(q), _p(xyz), _p(q), rows[0], rows[1], cols[0],
                                    cols[1], _p(out)))
    return out


def exp_glibc_host(x):
    """The device exp restatement (common.cuh exp_glibc_core) run on the host."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros_like(x)
    lib().h2g_exp_glibc_host(x.size, _p(x), _p(y))
    return y


def basis_from_members(concat, offsets, tol, cap=None, min_rank=0, qr_mode="exact"):
    concat = np.asfortranarray(concat, dtype=np.float64)
    dim = concat.shape[0]
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    sq = np.zeros((dim, dim), order="F")
    rank = np.zeros(1, dtype=np.int64)
    _check(lib().h2g_basis_from_members_mode(dim, concat.shape[1], _p(concat), len(offsets) - 1,
                                             _p(offsets), tol, cap or 0, min_rank,
                                             {"exact": 0, "blocked": 1, "compressed": 2}[qr_mode],
                                             _p(sq), _p(rank)))
    return sq, int(rank[0])
