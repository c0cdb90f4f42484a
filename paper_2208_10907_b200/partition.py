"""Multi-GPU partition of the level-parallel H2-ULV (host logic).

Ownership follows the reference's offline plan (partition_plan_json,
report.cpp:245-296): P = 2^p processes own contiguous leaf ranges; a box at
level l >= p belongs to rank (box >> (l - p)); levels < p are replicated
(the paper's tree-gather). On top of that plan this module
computes, per level, the halo each rank must receive before it can run its
dependency-free level stage on its own boxes:

  * near partners owned elsewhere: their diagonal LU (fills, solve
    row-combination) and near blocks A_pj (fill products W_pj);
  * far partners owned elsewhere: their shared bases (far skeletons S^SS);
  * at the replication level: an all-gather of the merged skeleton system.

send/recv lists are symmetric by construction (the block structure is
symmetric), which tests/test_partition.py checks across a gloo world.
"""
from dataclasses import dataclass, field
from typing import Dict, List, Tuple


def plan_levels(processes: int) -> int:
    if processes < 1 or processes & (processes - 1):
        raise ValueError("partition_plan: processes must be a power of two <= leaf count")
    p = 0
    while (1 << p) < processes:
        p += 1
    return p


def owner(level: int, box: int, plevels: int) -> int:
    """Rank owning box at level (or -1 when the level is replicated)."""
    if level < plevels:
        return -1
    return box >> (level - plevels)


@dataclass
class LevelHalo:
    level: int
    owned: List[int]
    recv_near: Dict[int, List[int]] = field(default_factory=dict)  # src rank -> boxes
    recv_far: Dict[int, List[int]] = field(default_factory=dict)
    send_near: Dict[int, List[int]] = field(default_factory=dict)  # dst rank -> boxes
    send_far: Dict[int, List[int]] = field(default_factory=dict)


def rank_plan(structure: Dict[int, Tuple], levels: int, processes: int, rank: int) -> List[LevelHalo]:
    """structure[lvl] = (near_ptr, near_idx, far_ptr, far_idx) (CSR, sorted)."""
    p = plan_levels(processes)
    if (1 << levels) < processes:
        raise ValueError("partition_plan: processes must be a power of two <= leaf count")
    out = []
    for lvl in range(levels, p - 1, -1):
        if lvl == 0:
            break
        nptr, nidx, fptr, fidx = structure[lvl]
        m = 1 << lvl
        owned = [i for i in range(m) if owner(lvl, i, p) == rank]
        h = LevelHalo(lvl, owned)
        for kind, ptr, idx, recv, send in (("near", nptr, nidx, h.recv_near, h.send_near),
                                           ("far", fptr, fidx, h.recv_far, h.send_far)):
            rset: Dict[int, set] = {}
            sset: Dict[int, set] = {}
            for i in owned:
                for t in range(ptr[i], ptr[i + 1]):
                    j = int(idx[t])
                    oj = owner(lvl, j, p)
                    if oj != rank:
                        rset.setdefault(oj, set()).add(j)
                        sset.setdefault(oj, set()).add(i)  # symmetric structure: j needs i
            for r, s in rset.items():
                recv[r] = sorted(s)
            for r, s in sset.items():
                send[r] = sorted(s)
        out.append(h)
    return out


def partition_plan(structure, levels, processes, ranks_by_level=None, cutoff_level=0):
    """h2ulv-partition-plan/1 (report.cpp:245-296) plus per-rank halo sizes."""
    p = plan_levels(processes)
    leaves = 1 << levels
    if processes > leaves:
        raise ValueError("partition_plan: processes must be a power of two <= leaf count")
    per = leaves // processes
    plan = {"schema": "h2ulv-partition-plan/1", "processes": processes, "leaves": leaves,
            "ownership": [{"process": r, "leaf_rows": [r * per, (r + 1) * per],
                           "leaf_cols": [r * per, (r + 1) * per]} for r in range(processes)],
            "replication_starts_at_level": p, "exchanges": []}
    for lvl in range(min(p, levels), 0, -1):
        nptr, nidx, fptr, fidx = structure[lvl]

        def rank_at(k):
            if ranks_by_level is None or lvl <= cutoff_level or lvl not in ranks_by_level:
                return 0
            return int(ranks_by_level[lvl][k])
        b = 0
        for i in range(1 << lvl):
            for t in range(nptr[i], nptr[i + 1]):
                b += rank_at(i) * rank_at(int(nidx[t])) * 8
            for t in range(fptr[i], fptr[i + 1]):
                b += rank_at(i) * rank_at(int(fidx[t])) * 8
        plan["exchanges"].append({"merge_to_level": lvl - 1, "exchanged_bytes": 0 if processes == 1 else b})
    return plan
