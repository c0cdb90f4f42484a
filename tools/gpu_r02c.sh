#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CAP=0 MODES=compressed timeout 900 python tools/corrected_scale.py 32768 65536 > gpurun_out/r02c_scale.jsonl 2> gpurun_out/r02c_scale.err
CAP=0 MODES=compressed COMPAT=1 timeout 900 python tools/corrected_scale.py 32768 65536 >> gpurun_out/r02c_scale.jsonl 2>> gpurun_out/r02c_scale.err
CAP=0 TOL=1e-7 MODES=blocked timeout 900 python tools/corrected_scale.py 32768 >> gpurun_out/r02c_scale.jsonl 2>> gpurun_out/r02c_scale.err
