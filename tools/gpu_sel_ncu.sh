O=gpurun_out
SEL_VARIANTS="- SIP_SELB_NS=3 SIP_SELB_NS=4" SEL_CONFIGS="C4" SEL_ITERS=2 bash tools/gpu_sel.sh 2>&1 | grep -v '^[-S].*ncand'
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_selB" --launch-skip 6 --launch-count 1 -f -o $O/s3_selB python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/s3_ncu_selB.log 2>&1; tail -1 $O/s3_ncu_selB.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_selC" --launch-skip 6 --launch-count 2 -f -o $O/s3_selC python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/s3_ncu_selC.log 2>&1; tail -1 $O/s3_ncu_selC.log
