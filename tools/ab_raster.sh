#!/bin/bash
# A/B of the raster record staging: cp.async (LDGSTS) vs cp.async.bulk (UBLKCP + mbarrier).
out=${1:-gpurun_out/ab}
mkdir -p $out
for rep in 1 2 3; do
  for v in 0 1; do
    GSIM_GPU_RASTER_BULK=$v python bench.py --steps 300 --no-cpu-baseline --no-e2e > $out/bulk${v}_$rep.log 2>&1
  done
done
for v in 0 1; do
  GSIM_GPU_RASTER_BULK=$v ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:raster -c 6 --csv \
    --log-file $out/ncu_bulk$v.csv python tools/profile_step.py --frames 3 > /dev/null 2>&1
done
