#!/bin/bash
# Round-end evidence run (TAG=r02p bash tools/gpu_evidence.sh): GPU tests, smoke, reference arm, bench, phase detail,
# ncu launch list and DRAM traffic of the GEMM kernels. Outputs under gpurun_out/${TAG}_*.
set -x
python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/${TAG:-rXX}_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG:-rXX}_smoke.log 2>&1
python bench.py > gpurun_out/${TAG:-rXX}_bench.json 2> gpurun_out/${TAG:-rXX}_bench.err
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/${TAG:-rXX}_reference_arm.json 2> gpurun_out/${TAG:-rXX}_reference_arm.err
python tools/prof_detail.py 65536 --warm > gpurun_out/${TAG:-rXX}_phase_detail.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${TAG:-rXX}_launches.csv python bench.py --steps 1 --warmup 1 --skip-cpu --exact-steps 0 --sampled-steps 0 --e2e-steps 1 > gpurun_out/${TAG:-rXX}_ncu_bench.log 2>&1
ncu --replay-mode application --kernel-name-base function --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k 'regex:gemm_p8_kernel|gemm_ws_kernel|gemm_kernel' --csv --log-file gpurun_out/${TAG:-rXX}_gemm_traffic.csv python tools/prof_detail.py 65536 > gpurun_out/${TAG:-rXX}_ncu_traffic.log 2>&1
tail -3 gpurun_out/${TAG:-rXX}_gputests.log
