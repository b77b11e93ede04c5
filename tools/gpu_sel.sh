#!/bin/bash
# select v2 A/B: k_selB candidate counts (SIP_SEL_DEBUG) and bench lines per
# variant ($SEL_VARIANTS: env settings, "-" = default), then an optional
# pytest -k subset
O=gpurun_out
VARS=${SEL_VARIANTS:-"- SIP_SEL_NOTSUM=1 SIP_SELC_FUSED=1"}
i=0
for v in $VARS; do
  E=$v; [ "$v" = "-" ] && E="SIP_NONE=0"
  env $E SIP_SEL_DEBUG=1 ITERS=${SEL_ITERS:-11} timeout 300 python tools/sel_debug.py 256x256x128 > $O/sel_dbg_$i.log 2>&1
  echo "$v: $(grep -o 'k=[0-9]* job=[0-9]* on_s=[0-9] kind=[0-9] mode=[0-9].*ncand=[0-9]*' $O/sel_dbg_$i.log | awk '{print $1,$3,$5,$NF}' | head -12 | tr '\n' ';')"
  i=$((i+1))
done
for c in ${SEL_CONFIGS:-C4 C5}; do
  s=10; [ $c = C5 ] && s=3
  i=0
  for v in $VARS; do
    E=$v; [ "$v" = "-" ] && E="SIP_NONE=0"
    env $E timeout 600 python bench.py --config $c --no-cpu-baseline --steps $s > $O/sel_bench_${c}_$i.json 2>&1
    echo "$c $v"; python tools/bench_brief.py $O/sel_bench_${c}_$i.json 2>&1 | grep -E '==|pass1|select'
    i=$((i+1))
  done
done
if [ -n "$PYTEST_K" ]; then env $PYTEST_ENV timeout 1500 python -m pytest tests -m gpu -q -k "$PYTEST_K" -p no:cacheprovider > $O/sel_pytest.log 2>&1; tail -8 $O/sel_pytest.log; fi
