#!/bin/bash
# Round r01e: GPU test suite, smoke, reference arm, then the bench evidence.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r01e_gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r01e_gputests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r01e_smoke.log 2>&1
python bench.py --impl reference > gpurun_out/r01e_ref.json 2> gpurun_out/r01e_ref.err
bash tools/prof_r01e.sh
