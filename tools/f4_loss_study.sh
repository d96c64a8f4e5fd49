#!/bin/bash
# k_fused4 per-row bound study: the same C2 shape with a closed-form prox (LS, hinge) vs the
# logistic Newton, FP64 and FP32, axpy delay 2 and 4.
OUT=${1:-gpurun_out/f4loss}
mkdir -p "$OUT"
for dt in f64 f32; do for loss in ls hinge logistic; do for D in 2 4; do
  BICADMM_F4_D=$D timeout 300 python bench.py --dtype $dt --loss $loss --steps 10 --warmup 3 --no-e2e --no-cpu --no-ttt \
    > "$OUT/${dt}_${loss}_d$D.json" 2> "$OUT/${dt}_${loss}_d$D.err"
  python - "$OUT/${dt}_${loss}_d$D.json" "$dt $loss D=$D" <<'PY'
import json, sys
d = json.load(open(sys.argv[1])); k = d["kernels"]
print(sys.argv[2], "sweeps/s %.1f" % d["config"]["sweeps_per_s"], "fused ms %.3f" % k["fused_sweep"]["ms_per_call"],
      "GB/s %.0f" % k["fused_sweep"]["GB_per_s"], "clk", d["clocks"]["sm_mhz"])
PY
done; done; done
