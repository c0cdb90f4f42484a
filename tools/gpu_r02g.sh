#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_corrected.py tests/test_bench_parity.py tests/test_multigpu.py > gpurun_out/r02g_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02g_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 --skip-cpu --exact-steps 0 > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
H2G_PROF_DETAIL=1 timeout 600 python tools/prof_detail.py 65536 --warm > gpurun_out/r02g_detail.txt 2>&1
