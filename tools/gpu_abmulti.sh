#!/bin/bash
# A/B of several builds of the library on one box: libsip.so (A) vs libsip_<name>.so for each name in $ALTS
O=gpurun_out
L=paper_1902_09699_b200
mkdir -p $O
cp $L/libsip.so /tmp/libsip_A.so
for rep in 1 2; do
  for arm in A $ALTS; do
    if [ $arm = A ]; then cp /tmp/libsip_A.so $L/libsip.so; else cp $L/libsip_$arm.so $L/libsip.so; fi
    for c in ${CONFIGS:-C4}; do
      args="--config $c --no-cpu-baseline --steps 10"
      case $c in C5*) args="--config $c --no-cpu-baseline --steps 3";; esac
      timeout 600 python bench.py $args > $O/ablib.log 2>&1
      python - "$arm" "$c" <<'PY' | tee -a $O/abmulti.txt
import json, sys
try:
    d = json.loads(open('gpurun_out/ablib.log').read().strip().splitlines()[-1])
    print(sys.argv[1], sys.argv[2], round(d['value'], 1), {k: round(v, 3) for k, v in d['kernel_ms_per_step'].items() if v})
except Exception as e:
    print(sys.argv[1], sys.argv[2], 'FAILED', e)
PY
    done
  done
done
cp /tmp/libsip_A.so $L/libsip.so
