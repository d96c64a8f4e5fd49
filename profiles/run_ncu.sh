#!/bin/bash
# ncu evidence for the bench step (run under gpurun, 1 GPU).  Each ncu command is
# preceded by the same command exiting 0 without ncu (B200_PROFILING.md rule).
#   launches.csv : every library launch of the bench command with its device time
#   prof.ncu-rep : --set full of the two per-sweep kernels (k_fused4 = the CTA-pair
#                  single-pass sweep, k_symv_tiles = the packed H-apply) in sweep 3
set -u
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-ttt"
$CMD > "$OUT/plain.log" 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:^(void )?(bic::)?k_' -c 5000 --csv \
    --log-file "$OUT/launches.csv" $CMD > "$OUT/ncu_launches.log" 2>&1
echo "ncu launches rc=$?"
$CMD > "$OUT/plain2.log" 2>&1 && \
ncu --set full --clock-control none --import-source on -k 'regex:k_fused4|k_symv_tiles' -s 4 -c 2 \
    -o "$OUT/prof" $CMD > "$OUT/ncu_full.log" 2>&1
echo "ncu full rc=$?"
