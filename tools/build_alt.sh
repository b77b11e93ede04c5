#!/bin/bash
# build paper_1902_09699_b200/libsip_alt.so with extra -D flags (for tools/gpu_ablib.sh)
R=$(cd "$(dirname "$0")/.." && pwd)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -Xptxas -O3 \
  -I $R/include "$@" -o $R/paper_1902_09699_b200/libsip_alt.so $R/paper_1902_09699_b200/csrc/sip_runtime.cu -lcublas
