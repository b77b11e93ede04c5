#!/bin/bash
# measurement pass: C4 bench, C5 bench, ncu launch list of C4, ncu full of the top CG kernels
O=gpurun_out
timeout 600 python bench.py > $O/bench_c4.log 2>&1; tail -c 2600 $O/bench_c4.log; echo
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c5.log 2>&1; tail -c 2000 $O/bench_c5.log; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1; tail -2 $O/ncu_launch.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_cg1f|k_cg2f" --launch-skip 40 --launch-count 2 -f -o $O/cgfull python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_cg.log 2>&1; tail -2 $O/ncu_cg.log
