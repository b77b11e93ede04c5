#!/bin/bash
# round-2 measurement: changed parity tests, bench lines of every config,
# the C4 launch list and an ncu --set full capture of the hot kernels
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
if [ -n "$PYTEST_K" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "$PYTEST_K" > $O/pytest_sel.log 2>&1; tail -8 $O/pytest_sel.log
fi
for c in ${BENCH_CFGS:-C4}; do
  args="--config ${c%%:*}"
  case $c in *:ml) args="$args --multilevel";; *:null) args="$args --null-work";; esac
  timeout 900 python bench.py $args --no-cpu-baseline ${BENCH_EXTRA} > $O/bench_${c/:/_}.json 2> $O/bench_${c/:/_}.err; tail -c 600 $O/bench_${c/:/_}.json; echo
done
if [ -n "$NCU_LIST" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_list.log 2>&1; tail -2 $O/ncu_list.log
fi
if [ -n "$NCU_K" ]; then
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"$NCU_K" --launch-skip ${NCU_SKIP:-40} --launch-count ${NCU_N:-8} -f -o $O/full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full.log 2>&1; tail -3 $O/ncu_full.log
fi
