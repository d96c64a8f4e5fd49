#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py (one tool per run).
# Usage (on the GPU box): bash tools/sanitize.sh gpurun_out/sanitize
OUT=${1:-gpurun_out/sanitize}
mkdir -p "$OUT"
CASES="fused4_g1 fused4_g2 fused4_g3 fused4_g4 fused4_g6 fused4_n2000 fused4_f32 gram_tc gemv_t_tma woodbury emu2"
for tool in memcheck racecheck synccheck initcheck; do
  for c in $CASES; do
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/sanitize_cases.py $c > "$OUT/${tool}_${c}.log" 2>&1
    echo "$tool $c rc=$?" | tee -a "$OUT/summary.txt"
  done
done
