#!/bin/bash
# Full evidence run on one B200: gpu tests, smoke, every bench workload, the
# launch list (ncu gpu__time_duration) of each, and one `ncu --set full`
# capture per kernel family. Output: gpurun_out/prof/ (copied to profiles/ by hand).
O=gpurun_out/prof
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt 2>&1
timeout -s KILL 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -5 > $O/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
for w in gemm_bf16 gemm_fp32 gemm_i8 attention attention_causal resnet50_convs bert_layer softmax layernorm; do
  timeout -s KILL 300 python bench.py --workload $w --steps 10 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err
done
for n in 2048 4096 8192; do
  timeout -s KILL 300 python bench.py --workload gemm_bf16 --size $n --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_gemm_bf16_$n.json 2>/dev/null
done
timeout -s KILL 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2>&1
# launch lists (cold-cache, serialised: shares, not absolutes)
for w in gemm_bf16 gemm_i8 attention attention_causal resnet50_convs bert_layer softmax layernorm gemm_fp32; do
  timeout -s KILL 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$w.csv \
    python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
done
# one full capture per kernel family (the dominant kernel of each workload)
cap() {  # workload kernel-regex tag [extra bench args]
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 -o $O/full_$3 \
    python bench.py --workload $1 --steps 1 --warmup 3 --no-cpu-baseline --no-graph $4 > $O/full_$3.log 2>&1
  # keep CSV exports only (gpurun copies back <= 64 MiB)
  ncu -i $O/full_$3.ncu-rep --page raw --csv > $O/full_$3_raw.csv 2>/dev/null
  ncu -i $O/full_$3.ncu-rep --page details --csv > $O/full_$3_details.csv 2>/dev/null
  ncu -i $O/full_$3.ncu-rep --page source --csv --print-source sass > $O/full_$3_sass.csv 2>/dev/null
  gzip -f $O/full_$3_sass.csv
  rm -f $O/full_$3.ncu-rep
}
cap gemm_bf16 gemm_tc gemm_bf16_16384
cap attention attn_fwd attention
cap attention_causal attn_fwd attention_causal
cap softmax stream_rows softmax
cap layernorm stream_rows layernorm
cap resnet50_convs conv_halo resnet_conv_halo
cap resnet50_convs gemm_tc resnet_conv_gemm
cap bert_layer attn_fwd bert_attention
cap gemm_fp32 gemm_simt gemm_fp32
cap gemm_i8 gemm_i8 gemm_i8_16384
echo done > $O/done
