#!/bin/bash
# k_fused4 axpy-delay sweep (BICADMM_F4_D) for FP64/FP32, logistic and LS prox, C2 shape.
OUT=${1:-gpurun_out/f4d2}
mkdir -p "$OUT"
DS=${DS:-"2 3 4 6 8"}
for dt in f32 f64; do for loss in logistic ls; do for D in $DS; do
  BICADMM_F4_D=$D timeout 300 python bench.py --dtype $dt --loss $loss --steps 10 --warmup 3 --no-e2e --no-cpu --no-ttt \
    > "$OUT/${dt}_${loss}_d$D.json" 2> "$OUT/${dt}_${loss}_d$D.err"
  python - "$OUT/${dt}_${loss}_d$D.json" "$dt $loss D=$D" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1])); k = d["kernels"]
    print(sys.argv[2], "sweeps/s %.1f" % d["config"]["sweeps_per_s"], "fused ms %.3f" % k["fused_sweep"]["ms_per_call"],
          "GB/s %.0f" % k["fused_sweep"]["GB_per_s"], "clk", d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done; done; done
