#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --workload resnet50_convs --only --steps 1 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/resnet_launches_all.csv 2>/dev/null
python - <<'PY'
import csv, io
txt = open("gpurun_out/resnet_launches_all.csv").read()
txt = txt[txt.index('"ID"'):]
rows = list(csv.reader(io.StringIO(txt)))
h = rows[0]
# keep the last 53 conv launches (the final step)
body = [r for r in rows[1:] if "fill" not in r[h.index("Kernel Name")]]
last = body[-53:]
with open("gpurun_out/resnet_launches.csv", "w") as f:
    f.write('"ID"' + txt[4:txt.index("\n")] + "\n")
    w = csv.writer(f, quoting=csv.QUOTE_ALL)
    for r in last: w.writerow(r)
PY
python scripts/conv_layers.py gpurun_out/resnet_launches.csv > gpurun_out/resnet_per_layer.txt 2>&1
cat gpurun_out/resnet_per_layer.txt
