#!/bin/bash
# A/B of libsip_fb9.so (k_selB's candidate histogram at 512 buckets: one k_selC round fewer) + the threshold-search tests on it
O=gpurun_out
L=paper_1902_09699_b200
mkdir -p $O
ALTS="fb9" CONFIGS="C4 C5 C2" bash tools/gpu_abmulti.sh
cp $L/libsip.so /tmp/libsip_A.so
cp $L/libsip_fb9.so $L/libsip.so
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_slabs.py -m gpu -q -p no:cacheprovider -k "project_set or tiny or c4 or c2 or c5 or fp32" > $O/pytest_fb9.log 2>&1; tail -5 $O/pytest_fb9.log
cp /tmp/libsip_A.so $L/libsip.so
