#!/bin/bash
# GPU check: the -m gpu suite (all failures listed), optional extra command
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout ${SUITE_TIMEOUT:-1800} python -m pytest tests -m gpu -q ${PYTEST_K:+-k "$PYTEST_K"} -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -30 $O/pytest_gpu.log
if [ -n "$EXTRA" ]; then bash -c "$EXTRA"; fi
