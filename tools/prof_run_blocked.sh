#!/bin/bash
# ncu evidence for the blocked-QR bench step (outputs under gpurun_out/):
#  1. launch list of one bench step (shares), 2. DRAM traffic of every qrb
#  launch of one factorization, 3. --set full of the longest qrb launch.
set -e
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_r01c.csv \
  python bench.py --steps 1 --warmup 0 --skip-cpu --exact-steps 0 > gpurun_out/ncu_launch_r01c.log 2>&1 || true
ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  -k regex:qrb_kernel --csv env H2G_QR_MODE=blocked python tools/prof_run.py 65536 > gpurun_out/qrb_traffic_r01c.csv 2>&1 || true
H2G_QR_MODE=blocked bash tools/ncu_top_launch.sh qrb_kernel qrb_r01c python tools/prof_run.py 65536 || true
