#!/bin/bash
# per-launch DRAM traffic (read + write) of each workload's dominant kernel,
# one ncu launch after warm-up, for profiles/traffic.json (bench roofline.traffic)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/traffic; o=gpurun_out/traffic/raw.txt; : > $o
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
run() {  # name, kernel regex, bench args
  local name=$1 k=$2; shift 2
  echo "== $name" >> $o
  timeout 600 ncu --metrics $M --clock-control none -k regex:$k -s 4 -c 1 python bench.py "$@" --only --no-cpu-baseline --steps 1 --warmup 4 --no-graph 2>/dev/null | grep -E "dram__|duration" >> $o
}
run gemm_bf16_gelu_16384 gemm_tc --size 16384
run gemm_bf16_gelu_8192 gemm_tc --size 8192
run gemm_bf16_gelu_4096 gemm_tc --size 4096
run gemm_bf16_gelu_2048 gemm_tc --size 2048
run gemm_splitk_16384 gemm_tc --workload gemm_splitk --size 16384
run gemm_i8_8192 gemm_i8 --workload gemm_i8 --size 8192
run gemm_fp32_relu gemm_f32 --workload gemm_fp32
run attention attn_fwd --workload attention
run attention_causal attn_fwd --workload attention_causal
run softmax stream_rows --workload softmax
run layernorm stream_rows --workload layernorm
cat $o
