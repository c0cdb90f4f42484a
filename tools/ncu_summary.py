"""Summarise ncu outputs into profiles/ (launch shares, per-kernel counters)."""
import csv
import collections
import json
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]
    ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0, 's': 1e3, 'second': 1e3}
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        name = r[ki].split('(')[0].replace('void ', '').replace('h2g::', '').replace('<unnamed>::', '')
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(',', '')) * scale.get(r[ui], 1.0)
    tot = sum(a[1] for a in agg.values())
    out = ["| kernel | launches | total ms (ncu, serialised) | share |", "|---|---|---|---|"]
    for k, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| {k} | {c} | {ms:.1f} | {100 * ms / tot:.1f}% |")
    return "\n".join(out), {k: v for k, v in agg.items()}


WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__grid_size', 'launch__block_size',
        'launch__registers_per_thread', 'launch__cluster_dim_x', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_tensor_op_dmma.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active',
        'lts__t_sector_hit_rate.pct', 'dram__throughput.avg.pct_of_peak_sustained_elapsed']


def raw(rep):
    txt = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    d = {}
    for w in WANT:
        if w in h:
            i = h.index(w)
            d[w] = (v[i], u[i])
    return d


if __name__ == '__main__':
    mode = sys.argv[1]
    if mode == 'launches':
        table, _ = launches(sys.argv[2])
        print(table)
    else:
        for k, (v, u) in raw(sys.argv[2]).items():
            print(f"| {k} | {v} {u} |")
