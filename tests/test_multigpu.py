"""Multi-GPU level partition (h2g_set_comm_*): box ownership follows the
reference's offline plan (partition_plan_json, report.cpp:245-296), and a
partitioned factorization reproduces the single-GPU factors bit for bit.

The GPU test runs two ranks as two processes on the one visible GPU with the
host-mediated exchange (gloo all-gather through pinned host buffers): the
ranks' kernels never wait on one another, only the host exchange joins them.
On an 8 x B200 node the same code path runs with h2g_set_comm_nccl."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2208_10907_b200 import _lib as g
from paper_2208_10907_b200 import partition


def test_partition_range_is_the_reference_plan():
    """h2g_partition_range == partition.owner (box >> (l - log2 P)) for every
    partitioned level; coarser levels are replicated."""
    for P in (1, 2, 4, 8):
        p = partition.plan_levels(P)
        for lvl in range(0, 9):
            m = 1 << lvl
            for r in range(P):
                lo, hi = g.partition_range(m, P, r)
                if P > 1 and lvl >= p:
                    assert [b for b in range(m) if partition.owner(lvl, b, p) == r] == list(range(lo, hi))
                else:
                    assert (lo, hi) == (0, m)


def test_partition_range_covers_ragged_levels():
    for P in (2, 3, 5, 8):
        for m in (P, P + 1, 37, 1000):
            spans = [g.partition_range(m, P, r) for r in range(P)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(spans[r][1] == spans[r + 1][0] for r in range(P - 1))
    with pytest.raises(g.H2GError):
        g.partition_range(4, 2, 2)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _solve(p, n):
    from oracle import ref
    b = ref.splitmix_signed(n, 7)
    return p.solve(b)


def _factor_case(case, comm=None):
    import paper_2208_10907_b200 as h2
    from oracle import cpu
    geom, n, leaf, kind, cap, tol = case[:6]
    mode = case[6] if len(case) > 6 else "exact"
    xyz, q = cpu.generate(geom, n, 42)
    p = h2.Problem()
    p.set_kernel(kind, 1.0 if kind == "yukawa" else 0.0, 1.0, 1e-3)
    p.set_options(tol=tol, cap=cap, qr_mode=mode)
    p.build(xyz, q, leaf)
    if comm is not None:
        p.set_comm(g.Comm.host(*comm, g.gloo_allgather()))
    p.factor()
    x = _solve(p, n)
    bases = [p.basis(p.levels, k, side)[0] for k in range(1 << p.levels) for side in (0, 1)]
    ranks = [rk.tolist() for _, rk in p.factor_levels()]
    p.close()
    return x, bases, ranks


def _worker(rank, world, port, case, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, bases, ranks = _factor_case(case, (world, rank))
        np.save(os.path.join(out, f"x{rank}.npy"), x)
        np.savez(os.path.join(out, f"b{rank}.npz"), *bases)
        np.save(os.path.join(out, f"r{rank}.npy"), np.array(sum(ranks, [])))
    finally:
        dist.destroy_process_group()


CASES = [("cube", 4096, 128, "laplace", 0, 1e-8),
         ("cube", 8192, 128, "laplace", 64, 1e-4),
         ("cube", 4096, 128, "laplace", 0, 1e-8, "blocked"),
         ("cube", 4096, 128, "laplace", 0, 1e-6, "compressed")]


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", CASES, ids=["c1_cube4096", "cube8192_cap64", "c1_cube4096_blockedqr",
                                         "cube4096_tol1e-6_compressedqr"])
def test_partitioned_factor_is_bitwise_single_gpu(tmp_path, world, case):
    x1, b1, r1 = _factor_case(case)
    mp.spawn(_worker, args=(world, _port(), case, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        xr = np.load(tmp_path / f"x{r}.npy")
        assert np.array_equal(xr.view(np.int64), x1.view(np.int64)), f"rank {r}: x differs"
        br = np.load(tmp_path / f"b{r}.npz")
        assert all(np.array_equal(br[f"arr_{i}"].view(np.int64), b.view(np.int64)) for i, b in enumerate(b1))
        assert np.load(tmp_path / f"r{r}.npy").tolist() == sum(r1, [])


@pytest.mark.gpu
def test_nccl_communicator_single_rank():
    """libnccl.so.2 resolves at run time and a 1-rank communicator is a no-op
    partition (the factors are the single-GPU ones)."""
    uid = g.nccl_unique_id()
    assert len(uid) == 128
    comm = g.Comm.nccl(1, 0, uid)
    x1, _, _ = _factor_case(CASES[0])
    import paper_2208_10907_b200 as h2
    from oracle import cpu
    xyz, q = cpu.generate("cube", 4096, 42)
    p = h2.Problem()
    p.set_kernel("laplace", 0.0, 1.0, 1e-3)
    p.set_options(tol=1e-8)
    p.build(xyz, q, 128)
    p.set_comm(comm)
    p.factor()
    x = _solve(p, 4096)
    p.close()
    comm.close()
    assert np.array_equal(x.view(np.int64), x1.view(np.int64))
