#!/bin/bash
# Round r01e evidence for the bench (compressed QR mode): bench line, launch
# list of one bench step, and the DRAM traffic of the dominant kernel family
# ("gemm": every gemm_ws_kernel<0> / gemm_kernel launch of one factorization).
set -x
python bench.py > gpurun_out/r01e_bench.json 2> gpurun_out/r01e_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    python bench.py --steps 1 --warmup 0 --skip-cpu --exact-steps 0 > gpurun_out/r01e_launches.csv 2> gpurun_out/r01e_launches.err
H2G_QR_MODE=compressed ncu --replay-mode application --kernel-name-base demangled \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    -k 'regex:gemm_ws_kernel<.int.0>|gemm_kernel' --csv python tools/prof_run.py 65536 \
    > gpurun_out/r01e_gemm_traffic.csv 2> gpurun_out/r01e_gemm_traffic.err
