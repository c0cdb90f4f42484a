#!/bin/bash
# Profiling pass: per-phase kernel detail, host-gap timeline, ncu launch list of the bench.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
H2G_PROF_DETAIL=1 timeout 600 python tools/prof_detail.py 65536 --warm > gpurun_out/r02f_detail.txt 2>&1
H2G_TIMELINE=1 timeout 600 python tools/prof_detail.py 65536 --warm > gpurun_out/r02f_timeline.txt 2> gpurun_out/r02f_timeline.err
timeout 900 python bench.py --steps 2 --warmup 1 --skip-cpu --exact-steps 0 --e2e-steps 1 > gpurun_out/r02f_bench_plain.json 2> gpurun_out/r02f_bench_plain.err
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r02f_launches.csv \
  python bench.py --steps 2 --warmup 1 --skip-cpu --exact-steps 0 --e2e-steps 1 > gpurun_out/r02f_ncu_bench.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r02f_ncu_bench.log
