#!/bin/bash
# round-2 final measurements: bench lines of every config, the C4 launch
# list, an ncu --set full capture of the hot kernels, the Fig. 1 experiment
# and smoke().  Writes gpurun_out/r2_*.
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/r2_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/r2_smoke.log 2>&1; tail -4 $O/r2_smoke.log
timeout 900 python bench.py > $O/r2_bench_C4.json 2> $O/r2_bench_C4.err
for c in C1 C1:null C2 C3 C5 C5:ml; do
  args="--config ${c%%:*} --no-cpu-baseline"
  case $c in *:ml) args="$args --multilevel";; *:null) args="$args --null-work";; esac
  case $c in C5*) args="$args --steps 3";; esac
  timeout 900 python bench.py $args > $O/r2_bench_${c/:/_}.json 2> $O/r2_bench_${c/:/_}.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/r2_bench_reference.json 2>&1
timeout 600 python tools/fig1_dykstra.py --out $O/r2_fig1_dykstra.json > $O/r2_fig1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/r2_launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/r2_ncu_list.log 2>&1
rm -f $O/r2_full*.ncu-rep
for k in k_cg1f k_cg2f k_pass1t k_rhsp k_selB k_selC k_pass2t k_cgx; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$k" --launch-skip 6 --launch-count 2 -f -o $O/r2_full_$k python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/r2_ncu_full_$k.log 2>&1
  tail -1 $O/r2_ncu_full_$k.log
done
# summaries are made here (the reports together can exceed gpurun_out's 64 MiB limit);
# reports are then dropped, largest first, until the directory fits
for f in $O/r2_full_*.ncu-rep; do
  python tools/ncu_summary.py $f > ${f%.ncu-rep}.summary.txt 2>&1
done
while [ $(du -sm $O | cut -f1) -ge 56 ]; do
  big=$(ls -S $O/*.ncu-rep 2>/dev/null | head -1); [ -z "$big" ] && break; rm -f $big
done
if [ -n "$SANITIZE" ]; then
  timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_case.py > $O/r2_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -5 $O/r2_memcheck.log
fi
