#!/bin/bash
# Round-2 ncu captures (run on the GPU box through gpurun; read with tools/summarise_profiles.py):
#   1. per-launch metrics of every heavy kernel of one cfg4 and one cfg5 search (time, DRAM bytes,
#      pipe utilisation, stall reasons) -> CSV
#   2. one `--set full` capture (with source) of the dominant kernel of each regime
set -u
OUT=gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"
M="$M,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"
M="$M,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active"
M="$M,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum"
for st in barrier long_scoreboard short_scoreboard math_pipe_throttle mio_throttle wait not_selected lg_throttle membar dispatch_stall no_instruction sleeping; do
  M="$M,smsp__average_warps_issue_stalled_${st}_per_issue_active.ratio"
done
HEAVY='regex:k_scan_tiles|k_bucket_mates|k_build_rows|k_window_encode4|k_seed_lower_bound|k_propagate|k_exact_nn|k_radix_scatter|k_gather_rows'
python tools/run_workload.py 4 5 > $OUT/r2_prof_plain.log 2>&1 || exit 1
ncu --metrics $M --clock-control none -k "$HEAVY" --csv --log-file $OUT/r2_metrics_cfg4.csv python tools/run_workload.py 4 > $OUT/r2_ncu_m4.log 2>&1
ncu --metrics $M --clock-control none -k "$HEAVY" --csv --log-file $OUT/r2_metrics_cfg5.csv python tools/run_workload.py 5 > $OUT/r2_ncu_m5.log 2>&1
# full captures: the 41st ws16 launch of cfg5 (a large window round of the first full batch); for cfg4 the
# 20th filter-kernel launch (the long tail of the second batch), and the three preparation / seeding kernels
ncu --set full --clock-control none --import-source on -k regex:k_scan_tiles_ws16 -s 24 -c 1 -f -o $OUT/r2_full_ws16_cfg5 python tools/run_workload.py 5 > $OUT/r2_ncu_f5.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_scan_tiles<" -s 19 -c 1 -f -o $OUT/r2_full_scanlb_cfg4 python tools/run_workload.py 4 > $OUT/r2_ncu_f4a.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_bucket_mates|k_build_rows|k_window_encode4|k_seed_lower_bound" -c 4 -f -o $OUT/r2_full_prep_cfg4 python tools/run_workload.py 4 > $OUT/r2_ncu_f4b.log 2>&1
ls -la $OUT/r2_full_*.ncu-rep $OUT/r2_metrics_*.csv
