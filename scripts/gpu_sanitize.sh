#!/bin/bash
# compute-sanitizer over the mbarrier / TMA pipelines (small shapes)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/sanitize
for tool in synccheck racecheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_probe.py \
    > gpurun_out/sanitize/$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize/$tool.txt
done
tail -n 5 gpurun_out/sanitize/*.txt
