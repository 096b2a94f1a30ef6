for g in 0 4 8 16 32; do echo group=$g; AFG_GEMM_GROUP_M=$g python scripts/gemm_probe.py 16384,16384,16384,3 8192,8192,8192,3; done
for g in 4 8 16; do AFG_GEMM_GROUP_M=$g timeout 120 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_tc -c 1 python scripts/gemm_probe.py 16384,16384,16384,3 2>&1 | grep -E "dram__bytes|duration" | sed "s/^/g=$g /"; done
