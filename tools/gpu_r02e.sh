#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python tools/explicit_ulv_gpu.py 16384 256 1e-6 100 0 > gpurun_out/r02e_explicit16k.log 2>&1
timeout 1500 python tools/explicit_ulv_gpu.py 32768 256 1e-6 100 0 > gpurun_out/r02e_explicit32k.log 2>&1
timeout 900 python -m pytest -q -m gpu tests/test_dropin.py tests/test_facade.py > gpurun_out/r02e_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02e_tests.log
