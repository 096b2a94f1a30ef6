#!/bin/bash
# ncu captures of the round-2 kernels (one GPU, one kernel each)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/prof
NCU="ncu --set full --import-source on --clock-control none"
timeout 600 $NCU -k regex:stream_rows -s 8 -c 1 -o gpurun_out/prof/layernorm python bench.py --workload layernorm --only --steps 3 --no-cpu-baseline --no-graph > gpurun_out/prof/ln.log 2>&1
timeout 600 $NCU -k regex:gemm_f32_8x8 -s 5 -c 1 -o gpurun_out/prof/gemm_fp32 python bench.py --workload gemm_fp32 --only --steps 3 --no-cpu-baseline --no-graph > gpurun_out/prof/fp32.log 2>&1
timeout 600 $NCU -k regex:nest_vm -c 1 -o gpurun_out/prof/nest_vm python scripts/vm_region_probe.py 2048 4096 > gpurun_out/prof/vm.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python bench.py --workload gemm_splitk --only --steps 3 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/prof/splitk_launches.csv 2>/dev/null
python scripts/vm_region_probe.py 2048 4096 > gpurun_out/prof/vm_time.txt 2>&1
for f in gpurun_out/prof/*.ncu-rep; do ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null; ncu -i $f --page details --csv > ${f%.ncu-rep}_details.csv 2>/dev/null; done
rm -f gpurun_out/prof/*.ncu-rep
ls -la gpurun_out/prof
