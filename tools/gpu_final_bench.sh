#!/bin/bash
# final benches of the round (after the test suite ran on its own): C4 bench
# with the CPU baseline, C5-L1, the reference arm, the ncu launch list and a
# full capture of the hot kernels
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/final_smoke.log 2>&1; cat $O/final_smoke.log
timeout 600 python bench.py > $O/final_bench_c4.log 2>&1; tail -c 3000 $O/final_bench_c4.log; echo
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > $O/final_bench_c5.log 2>&1; tail -c 600 $O/final_bench_c5.log; echo
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/final_bench_ref.log 2>&1; tail -c 400 $O/final_bench_ref.log; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/final_launches_c4.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/final_ncu_launch.log 2>&1; tail -1 $O/final_ncu_launch.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_cg1f|k_cg2f|k_selectf|k_pass1t|k_rhsf|k_pass2t|k_cgx|k_initv" --launch-skip 60 --launch-count 14 -f -o $O/final_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/final_ncu_full.log 2>&1; tail -1 $O/final_ncu_full.log
