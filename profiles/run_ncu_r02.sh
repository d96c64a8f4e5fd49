#!/bin/bash
# Round-2 ncu evidence (run under gpurun, 1 GPU).  Each ncu command is preceded by the same
# command exiting 0 without ncu (B200_PROFILING.md rule).
#   launches_<dt>.csv : every library launch of the bench command with its device time
#   full_<dt>.ncu-rep : --set full of the per-sweep kernels (k_fused4 single-pass sweep,
#                       k_symv_tiles packed H-apply) in sweep 4
set -u
OUT=${1:-gpurun_out/ncu_r02}
mkdir -p "$OUT"
for dt in f64 f32; do
  CMD="python bench.py --dtype $dt --steps 2 --warmup 3 --no-e2e --no-cpu --no-ttt"
  $CMD > "$OUT/plain_$dt.log" 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:^(void )?(bic::)?k_' -c 5000 --csv \
      --log-file "$OUT/launches_$dt.csv" $CMD > "$OUT/ncu_launches_$dt.log" 2>&1
  echo "$dt ncu launches rc=$?"
  ncu --set full --clock-control none --import-source on -k 'regex:k_fused4|k_symv_tiles' -s 4 -c 2 \
      -o "$OUT/full_$dt" $CMD > "$OUT/ncu_full_$dt.log" 2>&1
  echo "$dt ncu full rc=$?"
done
