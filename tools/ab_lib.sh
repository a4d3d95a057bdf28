# A/B(/C...) builds of libgsim_gpu.so on one box:
#   bash tools/ab_lib.sh ROUNDS LIB1 LIB2 [LIB3 ...] -- [bench args]
# Runs the default bench with each library in turn, ROUNDS times (L1 L2 L3 L1 L2 L3 ...), and
# prints value / e2e / stage times per run; the last library stays in place.
R=$1; shift
LIBS=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do LIBS+=("$1"); shift; done
[ "$1" = "--" ] && shift
mkdir -p gpurun_out
LIB=paper_2507_21981_b200/libgsim_gpu.so
for i in $(seq "$R"); do
  for v in "${LIBS[@]}"; do
    cp "$v" $LIB
    timeout 300 python bench.py "$@" 2>/dev/null | python -c "
import json, sys
d = json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('$(basename "$v")', d['value'], d['e2e']['value'], d['roofline']['stages_ms'], d.get('first_frame_hash'))"
  done
done
