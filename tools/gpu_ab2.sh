#!/bin/bash
# A/B bench (B_ENV) + ncu capture of kernels matching $NCU_K
O=gpurun_out
bash tools/gpu_ab.sh
if [ -n "$NCU_K" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$NCU_K --launch-skip ${NCU_SKIP:-20} --launch-count ${NCU_N:-2} -f -o $O/q python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_q.log 2>&1; tail -2 $O/ncu_q.log
fi
