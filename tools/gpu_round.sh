#!/bin/bash
# one GPU validation + measurement pass (run through gpurun from the repo root)
set -x
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_slabs.py -x -q > $O/pytest_slabs.log 2>&1; tail -5 $O/pytest_slabs.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -5 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench.log 2>&1; tail -c 600 $O/bench.log
timeout 600 python bench.py --virtual-ranks 8 --no-cpu-baseline --steps 5 > $O/bench_v8.log 2>&1; tail -c 900 $O/bench_v8.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; cat $O/smoke.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pass1t --launch-skip 4 --launch-count 2 -f -o $O/pass1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_pass1.log 2>&1; tail -3 $O/ncu_pass1.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_cg1z --launch-skip 20 --launch-count 1 -f -o $O/cg1z python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_cg1z.log 2>&1; tail -3 $O/ncu_cg1z.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_selectf --launch-skip 6 --launch-count 3 -f -o $O/select python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_select.log 2>&1; tail -3 $O/ncu_select.log
ls -la $O
