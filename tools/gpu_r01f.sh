#!/bin/bash
# Round r01f: GPU tests + bench after the chunked Lloyd chains and the
# handle-reusing e2e loop.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r01f_gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r01f_gputests.log
python bench.py > gpurun_out/r01f_bench.json 2> gpurun_out/r01f_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    python bench.py --steps 1 --warmup 0 --skip-cpu --exact-steps 0 --e2e-steps 1 > gpurun_out/r01f_launches.csv 2> gpurun_out/r01f_launches.err
