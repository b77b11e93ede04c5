O=gpurun_out; mkdir -p $O
timeout 900 python bench.py --config C1 --no-cpu-baseline > $O/sc_C1.json 2>$O/sc_C1.err; tail -c 300 $O/sc_C1.json; echo
SIP_NO_SMALL_CG=1 timeout 900 python bench.py --config C1 --no-cpu-baseline > $O/sc_C1_off.json 2>&1; tail -c 300 $O/sc_C1_off.json; echo
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "parity or fibers or canary or tiny or small or C1 or c1 or dykstra or dct or svd" > $O/pytest_sc.log 2>&1; tail -8 $O/pytest_sc.log
