#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py (GPU box).
#   bash tools/sanitize.sh [outdir]
out=${1:-gpurun_out/sanitize}
mkdir -p "$out"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for case in smoke copies contexts batch; do
    extra=""
    [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
    timeout 900 $CS --tool $tool $extra --error-exitcode 99 python tools/sanitize_cases.py $case \
      > "$out/${tool}_${case}.log" 2>&1
    echo "$tool $case exit=$?" | tee -a "$out/summary.txt"
  done
done
