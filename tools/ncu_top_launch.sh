#!/bin/bash
# Usage: tools/ncu_top_launch.sh <kernel-regex> <out-name> <cmd...>
# Lists the kernel's launches (duration only), then captures --set full of the
# longest one. Outputs under gpurun_out/.
set -e
re=$1; out=$2; shift 2
base=${NCU_NAME_BASE:-function}  # demangled: match template arguments, e.g. "gemm_ws_kernel<1>"
ncu --kernel-name-base $base --metrics gpu__time_duration.sum --clock-control none -k "regex:$re" --csv "$@" > gpurun_out/${out}_list.csv 2>/dev/null || true
idx=$(python3 - "$out" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/{sys.argv[1]}_list.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
t = [float(r[vi].replace(",", "")) for r in rows[1:]]
print(max(range(len(t)), key=lambda i: t[i]))
PY
)
echo "longest launch index $idx"
ncu --kernel-name-base $base --set full --clock-control none --import-source on -k "regex:$re" --launch-skip $idx -c 1 -o gpurun_out/$out "$@" > gpurun_out/${out}.log 2>&1
