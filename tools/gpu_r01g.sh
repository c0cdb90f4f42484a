#!/bin/bash
# Round r01g: final confirmation of HEAD from a fresh container build —
# GPU tests, smoke(), reference arm, default bench line.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r01g_gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r01g_gputests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r01g_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r01g_smoke.log
python bench.py --impl reference > gpurun_out/r01g_reference_arm.json 2> gpurun_out/r01g_reference_arm.err
python bench.py > gpurun_out/r01g_bench.json 2> gpurun_out/r01g_bench.err
echo done
