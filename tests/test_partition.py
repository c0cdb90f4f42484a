"""Multi-GPU partition host logic: ownership, halos and the reference's
partition plan; send/recv symmetry checked across a gloo world of 2."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cpu
from paper_2208_10907_b200 import partition


def structure(n=4096, leaf=64, seed=5):
    xyz, q = cpu.generate("cube", n, seed)
    _, _, _, _, geo, L = cpu.build_tree(xyz, q, leaf)
    return cpu.classify(L, geo), L


def test_ownership_partitions_every_box():
    s, L = structure()
    for P in (1, 2, 4, 8):
        p = partition.plan_levels(P)
        for lvl in range(max(p, 1), L + 1):
            owned = sorted(sum((h.owned for r in range(P)
                                for h in partition.rank_plan(s, L, P, r) if h.level == lvl), []))
            assert owned == list(range(1 << lvl))


def test_plan_schema_and_errors():
    s, L = structure()
    plan = partition.partition_plan(s, L, 4)
    assert plan["schema"] == "h2ulv-partition-plan/1" and plan["replication_starts_at_level"] == 2
    assert plan["ownership"][1]["leaf_rows"] == [(1 << L) // 4, 2 * (1 << L) // 4]
    with pytest.raises(ValueError):
        partition.partition_plan(s, L, 3)


def _worker(rank, world, port, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s, L = structure()
    mine = partition.rank_plan(s, L, world, rank)
    allp = [None] * world
    dist.all_gather_object(allp, [(h.level, h.owned, h.recv_near, h.send_near, h.recv_far, h.send_far)
                                  for h in mine])
    ok = True
    for lv in range(len(mine)):
        for r in range(world):
            for o in range(world):
                if r == o:
                    continue
                lvl_r = allp[r][lv]
                lvl_o = allp[o][lv]
                # what r receives from o equals what o sends to r
                ok &= lvl_r[2].get(o, []) == lvl_o[3].get(r, [])
                ok &= lvl_r[4].get(o, []) == lvl_o[5].get(r, [])
    result[rank] = ok
    dist.destroy_process_group()


def test_halo_symmetry_gloo_world2():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_worker, args=(2, port, result), nprocs=2, join=True)
    assert result[0] and result[1]
