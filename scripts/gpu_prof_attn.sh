#!/bin/bash
# ncu --set full + SASS stall sampling of the attention kernel (non-causal, causal)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/prof_attn
NCU="ncu --set full --import-source on --clock-control none"
for wl in attention attention_causal; do
  timeout 600 $NCU -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/prof_attn/$wl -f python bench.py --workload $wl --only --steps 1 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/prof_attn/$wl.log 2>&1
done
for f in gpurun_out/prof_attn/*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > ${b}_raw.csv 2>/dev/null
  ncu -i $f --page details --csv > ${b}_details.csv 2>/dev/null
  ncu -i $f --page source --csv --print-source sass > ${b}_sass.csv 2>/dev/null || ncu -i $f --page source --csv > ${b}_sass.csv 2>/dev/null
  gzip -f ${b}_sass.csv ${b}_raw.csv
done
rm -f gpurun_out/prof_attn/*.ncu-rep
ls -la gpurun_out/prof_attn
