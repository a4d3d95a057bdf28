# On the GPU box: ncu evidence for one config, summarised afterwards here with
#   python tools/summarize_profiles.py --tag r2_<cfg> --config <cfg> \
#       --launches gpurun_out/prof/launches_<cfg>.csv --report gpurun_out/prof/frame_<cfg>.ncu-rep
# 1) launch list (time + DRAM bytes per launch) of a short single-context bench run;
# 2) one `--set full` capture of every kernel of one frame (after two warm-up frames).
cfg=${1:-cfg1}
mkdir -p gpurun_out/prof
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/prof/launches_$cfg.csv \
    python bench.py --config $cfg --steps 4 --warmup 3 --contexts 1 --no-e2e --no-cpu-baseline \
    > gpurun_out/prof/launches_$cfg.log 2>&1
echo "launches $cfg exit=$?"
K='regex:^(void )?(gsim_gpu::)?(preprocess_kernel|key_hist_kernel|chunk_table_kernel|onesweep_kernel|bin_count_kernel|bin_colscan_kernel|bin_tilescan_kernel|bin_campre_kernel|bin_scatter_kernel|raster_kernel)'
timeout 1500 ncu --set full --import-source on --clock-control none -k "$K" --launch-skip 26 \
    --launch-count 13 -f -o gpurun_out/prof/frame_$cfg python tools/profile_step.py --config $cfg \
    --frames 1 --warmup 2 > gpurun_out/prof/frame_$cfg.log 2>&1
echo "frame $cfg exit=$?"
