#!/bin/bash
# Round-2 first GPU pass: corrected mode, glibc-exp Yukawa, benched-config parity, bench.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_gpu.txt 2>&1
timeout 1500 python -m pytest -x -q -m gpu tests/test_corrected.py tests/test_bench_parity.py \
  "tests/test_gpu_parity.py::test_yukawa_bitwise_vs_reference" > gpurun_out/r02a_newtests.log 2>&1
echo "newtests rc=$?" >> gpurun_out/r02a_newtests.log
timeout 1800 python -m pytest -q -m gpu tests > gpurun_out/r02a_gputests.log 2>&1
echo "gputests rc=$?" >> gpurun_out/r02a_gputests.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
echo "bench rc=$?" >> gpurun_out/r02a_bench.err
