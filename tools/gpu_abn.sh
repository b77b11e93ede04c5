#!/bin/bash
# A/B bench on one box over several configs, alternating A / B twice:
#   CONFIGS="C4 C5" B_ENV="SIP_X=1" [A_ENV=...] [PYTEST_K=...] bash tools/gpu_abn.sh
O=gpurun_out
mkdir -p $O
for rep in 1 2; do
for c in ${CONFIGS:-C4}; do
  args="--config ${c%%:*} --no-cpu-baseline --steps ${STEPS:-10}"
  case $c in *:ml) args="$args --multilevel";; esac
  case $c in C5*) args="$args --steps 3";; esac
  for arm in A B; do
    if [ $arm = A ]; then E="${A_ENV:-SIP_AB_NONE=1}"; else E="$B_ENV"; fi
    env $E timeout 600 python bench.py $args > $O/ab_${arm}_${c/:/_}.log 2>&1
    python - "$arm" "$c" "$O/ab_${arm}_${c/:/_}.log" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
    print(sys.argv[1], sys.argv[2], round(d['value'], 1), {k: round(v, 3) for k, v in d['kernel_ms_per_step'].items() if v})
except Exception as e:
    print(sys.argv[1], sys.argv[2], 'FAILED', open(sys.argv[3]).read()[-600:])
PY
  done
done
done
if [ -n "$PYTEST_K" ]; then timeout 1500 python -m pytest tests -m gpu -x -q -k "$PYTEST_K" -p no:cacheprovider > $O/pytest_ab.log 2>&1; tail -5 $O/pytest_ab.log; fi
