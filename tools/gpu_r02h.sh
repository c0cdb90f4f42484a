#!/bin/bash
# Fresh-container re-check of HEAD: full GPU suite, smoke, bench.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 2400 python -m pytest -q -m gpu tests > gpurun_out/r02h_gputests.log 2>&1
echo "gputests rc=$?" >> gpurun_out/r02h_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r02h_smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err
echo "bench rc=$?" >> gpurun_out/r02h_bench.err
