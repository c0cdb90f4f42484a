#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python tools/corrected_scale.py 16384 32768 65536 > gpurun_out/r02b_scale.jsonl 2> gpurun_out/r02b_scale.err
CAP=200 MODES=compressed timeout 900 python tools/corrected_scale.py 32768 65536 >> gpurun_out/r02b_scale.jsonl 2>> gpurun_out/r02b_scale.err
timeout 900 python -m pytest -q -m gpu tests/test_bench_parity.py tests/test_corrected.py tests/test_qr_blocked.py > gpurun_out/r02b_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02b_tests.log
