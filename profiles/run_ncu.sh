#!/bin/bash
# ncu evidence for the bench step (run under gpurun, 1 GPU).  Each ncu command is
# preceded by the same command exiting 0 without ncu (B200_PROFILING.md rule).
set -u
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-ttt"
KREGEX='regex:k_gemv|k_prox|k_zt|k_s_update|k_u_update|k_node_sq|k_residuals|k_wsum'
$CMD > "$OUT/plain.log" 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k "$KREGEX" --csv \
    --log-file "$OUT/launches.csv" $CMD > "$OUT/ncu_launches.log" 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 4 -c 4 \
    -o "$OUT/prof_gemv" $CMD > "$OUT/ncu_full.log" 2>&1
echo "ncu rc=$?"
