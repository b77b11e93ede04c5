#!/bin/bash
# GPU check: full -m gpu suite, bench, and an ncu capture of kernels matching $NCU_K
O=gpurun_out
set -x
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu.log 2>&1; tail -15 $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench.log 2>&1; tail -c 1400 $O/bench.log
if [ -n "$NCU_K" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$NCU_K --launch-skip ${NCU_SKIP:-4} --launch-count ${NCU_N:-2} -f -o $O/q python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_q.log 2>&1; tail -3 $O/ncu_q.log
fi
