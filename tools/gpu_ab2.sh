#!/bin/bash
# A/B on one box: libsip.so (B) vs libsip_ab.so (A), configs $CFGS, alternated twice
O=gpurun_out; mkdir -p $O
for rep in 1 2; do
for c in ${CFGS:-C4}; do
  SIP_LIBPATH=$PWD/paper_1902_09699_b200/libsip_ab.so timeout 600 python bench.py --config $c --no-cpu-baseline $BENCH_EXTRA > $O/ab_A_${c}_$rep.json 2>/dev/null
  timeout 600 python bench.py --config $c --no-cpu-baseline $BENCH_EXTRA > $O/ab_B_${c}_$rep.json 2>/dev/null
  python - $c $rep <<'PY'
import json,sys
c,rep=sys.argv[1:]
for s in 'AB':
    d=json.loads(open(f'gpurun_out/ab_{s}_{c}_{rep}.json').read().strip().splitlines()[-1])
    print(s, c, rep, round(d['value'],1), {k: round(v,3) for k,v in d['kernel_ms_per_step'].items() if v})
PY
done; done
if [ -n "$PYTEST_K" ]; then timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$PYTEST_K" > $O/pytest_ab.log 2>&1; tail -5 $O/pytest_ab.log; fi
