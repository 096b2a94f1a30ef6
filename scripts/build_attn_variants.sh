#!/bin/bash
# A/B builds of the attention kernel: libafg variants differing only in
# attention.cu's compile-time knobs, loaded with AFG_LIB_PATH.
# usage: build_attn_variants.sh name:"-DX=1 -DY=2" ...
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants variants
NV="/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude -cudart static"
OTHERS=$(ls build/afg/*.o | grep -v attention.o)
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  $NV $defs -Xptxas -v -c paper_2603_06731_b200/csrc/attention.cu -o build/variants/attention_$name.o 2> build/variants/attention_$name.ptxas.log
  echo "$name: $(grep -A2 "attn_fwd_kernelILi128ELb0" build/variants/attention_$name.ptxas.log | grep -E "spill|registers" | tr '\n' ' ')"
  $NV -shared -cudart static -o variants/libafg_$name.so build/variants/attention_$name.o $OTHERS -Xcompiler -fvisibility=hidden -ldl -lpthread
done
