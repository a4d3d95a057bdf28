#!/bin/bash
# Stand-in for compute-sanitizer (closed on the GPU pool): the GSIM_DCHECK bounds-checked library
# (libgsim_gpu_debug.so, common.cuh) over the sanitizer cases, the full-size parity tests and the
# mixed-camera scatter test, plus a run-to-run determinism check with concurrent contexts.
#   bash tools/debug_checks.sh [outdir]
out=${1:-gpurun_out/debug_checks}
mkdir -p "$out"
export GSIM_GPU_LIB=libgsim_gpu_debug.so
for case in smoke copies contexts batch determinism; do
  timeout 900 python tools/sanitize_cases.py $case > "$out/$case.log" 2>&1
  echo "dcheck $case exit=$?" | tee -a "$out/summary.txt"
done
timeout 1800 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_scene_stream.py tests/test_gpu_parity.py \
  -m gpu -q -x > "$out/pytest_debug.log" 2>&1
echo "dcheck pytest exit=$?" | tee -a "$out/summary.txt"
grep -h "GSIM_DCHECK failed" "$out"/*.log | sort | uniq -c | tee -a "$out/summary.txt"
