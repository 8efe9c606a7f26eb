#!/bin/bash
# Round-2 (second half) ncu captures, after the tensor-core tile kernel became the default for the dot form and for
# the tails of covering scans.  Run on the GPU box through gpurun; read with tools/summarise_profiles.py.
#   1. launch lists (gpu__time_duration.sum) of one search of cfg3, cfg4, cfg5
#   2. per-launch metrics of every heavy kernel of cfg4 and cfg5
#   3. `--set full` captures (with source): k_scan_tiles_tc on cfg5 (a large window round) and on cfg4 (a tail),
#      k_bucket_mates_runs / k_window_encode4 / k_build_rows on cfg4
set -u
OUT=gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"
M="$M,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"
M="$M,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"
M="$M,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active"
M="$M,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,lts__t_sector_hit_rate.pct"
for st in barrier long_scoreboard short_scoreboard math_pipe_throttle mio_throttle wait not_selected lg_throttle membar dispatch_stall no_instruction sleeping; do
  M="$M,smsp__average_warps_issue_stalled_${st}_per_issue_active.ratio"
done
HEAVY='regex:k_scan_tiles|k_bucket_mates|k_build_rows|k_window_encode4|k_seed_lower_bound|k_propagate|k_exact_nn|k_radix_scatter|k_gather_rows|k_split'
python tools/run_workload.py 3 4 5 > $OUT/r2b_prof_plain.log 2>&1 || exit 1
for c in 3 4 5; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r2b_launches_cfg$c.csv python tools/run_workload.py $c > $OUT/r2b_ncu_l$c.log 2>&1
done
ncu --metrics $M --clock-control none -k "$HEAVY" --csv --log-file $OUT/r2b_metrics_cfg4.csv python tools/run_workload.py 4 > $OUT/r2b_ncu_m4.log 2>&1
ncu --metrics $M --clock-control none -k "$HEAVY" --csv --log-file $OUT/r2b_metrics_cfg5.csv python tools/run_workload.py 5 > $OUT/r2b_ncu_m5.log 2>&1
# the 56th tensor-core launch of cfg5 is a wide window round of the first full batch; the 20th of cfg4 a tail of the second batch
ncu --set full --clock-control none --import-source on -k regex:k_scan_tiles_tc -s 55 -c 1 -f -o $OUT/r2b_full_tc_cfg5 python tools/run_workload.py 5 > $OUT/r2b_ncu_f5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_scan_tiles_tc -s 4 -c 1 -f -o $OUT/r2b_full_tc_cfg4 python tools/run_workload.py 4 > $OUT/r2b_ncu_f4.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_bucket_mates|k_build_rows|k_window_encode4|k_seed_lower_bound" -c 5 -f -o $OUT/r2b_full_prep_cfg4 python tools/run_workload.py 4 > $OUT/r2b_ncu_f4b.log 2>&1
ls -la $OUT/r2b_full_*.ncu-rep $OUT/r2b_metrics_*.csv $OUT/r2b_launches_*.csv
