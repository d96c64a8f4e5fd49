#!/bin/bash
# ncu --set full of the dominant kernels of the other per-GPU configs (1 GPU, one command
# each, each preceded by the same command exiting 0 without ncu):
#   C4  (softmax C = 10, M = 8, 80 GB): k_gemv_t_dmma_tma, k_gemv_dmma
#   C3s (LS, 1M x 12.5k, 100 GB, single pass): k_fused4
#   C5s (hinge, 8 x 250k x 6.25k, 100 GB, single pass): k_fused4
set -u
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
run() {   # name, kernel regex, launch skip, bench args
  local name=$1 kre=$2 skip=$3; shift 3
  local CMD="python bench.py $* --steps 1 --warmup 1 --no-e2e --no-cpu --no-ttt"
  $CMD > "$OUT/plain_$name.log" 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:$kre" -s "$skip" -c 2 \
      -o "$OUT/prof_$name" $CMD > "$OUT/ncu_$name.log" 2>&1
  echo "$name ncu rc=$?"
}
ONLY=${ONLY:-c4t c4 c3s c5s}
for cfg in $ONLY; do case $cfg in
  c4t) run c4t 'k_gemv_t_dmma' 1 --config C4 ;;
  c4) run c4 'k_gemv_dmma' 4 --config C4 ;;
  c3s) run c3s 'k_fused4' 2 --config C3s ;;
  c5s) run c5s 'k_fused4' 2 --config C5s ;;
esac; done
exit 0
run c3s 'k_gemv_t_partial|k_gemv<' 4 --config C3s
run c5s 'k_fused4' 2 --config C5s
