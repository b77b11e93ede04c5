#!/bin/bash
# A/B bench on one box: default vs env $B_ENV (e.g. SIP_NO_CGS=1), then optional pytest -k $PYTEST_K
O=gpurun_out
python bench.py --no-cpu-baseline --steps 10 > $O/bench_a.log 2>&1; python - <<'PY'
import json; d=json.loads(open('gpurun_out/bench_a.log').read().strip().splitlines()[-1]); print('A', round(d['value'],1), {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})
PY
env $B_ENV python bench.py --no-cpu-baseline --steps 10 > $O/bench_b.log 2>&1; python - <<'PY'
import json; d=json.loads(open('gpurun_out/bench_b.log').read().strip().splitlines()[-1]); print('B', round(d['value'],1), {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})
PY
if [ -n "$PYTEST_K" ]; then timeout 1500 python -m pytest tests -m gpu -x -q -k "$PYTEST_K" > $O/pytest_gpu.log 2>&1; tail -5 $O/pytest_gpu.log; fi
