#!/bin/bash
# A/B builds of the attention kernel: libafg variants differing only in
# attention.cu's compile-time knobs (loaded with AFG_LIB_PATH)
set -e
cd "$(dirname "$0")/.."
NV="/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude -cudart static"
OTHERS=$(ls build/afg/*.o | grep -v attention.o)
for pp in "$@"; do
  $NV -DAFG_POLY_PAIRS=$pp -Xptxas -v -c paper_2603_06731_b200/csrc/attention.cu -o build/variants/attention_$pp.o 2> build/variants/attention_$pp.ptxas.log
  grep -A2 "attn_fwd_kernelILi128ELb0" build/variants/attention_$pp.ptxas.log | grep spill | head -1
  $NV -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o variants/libafg_poly$pp.so build/variants/attention_$pp.o $OTHERS -Xcompiler -fvisibility=hidden -ldl -lpthread
done
