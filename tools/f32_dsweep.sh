#!/bin/bash
# FP32 single-pass sweep: axpy delay D and ring depth study at configs[1] (C2 shape, FP32 storage).
OUT=${1:-gpurun_out/f32d}
mkdir -p "$OUT"
for D in 2 3 4 5 6 7; do
  BICADMM_F4_D=$D timeout 300 python bench.py --dtype f32 --steps 10 --warmup 3 --no-e2e --no-cpu --no-ttt \
    > "$OUT/d$D.json" 2> "$OUT/d$D.err"
  python - "$OUT/d$D.json" $D <<'PY'
import json, sys
d = json.load(open(sys.argv[1])); k = d["kernels"]
print("D", sys.argv[2], "sweeps/s %.1f" % d["config"]["sweeps_per_s"], "fused ms %.3f" % k["fused_sweep"]["ms_per_call"],
      "GB/s %.0f" % k["fused_sweep"]["GB_per_s"], "h_apply ms %.3f" % k["h_apply"]["ms_per_call"], "clk", d["clocks"]["sm_mhz"])
PY
done
