#!/bin/bash
# compute-sanitizer passes over every kernel (tools/sanitize_workload.py); run on a GPU box:
#   bash tools/sanitize.sh [outdir]
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize_workload.py > "$OUT/sanitize_$tool.log" 2>&1
  echo "$tool rc=$?" >> "$OUT/sanitize_$tool.log"
  tail -2 "$OUT/sanitize_$tool.log"
done
