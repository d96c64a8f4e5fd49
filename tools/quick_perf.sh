#!/bin/bash
# quick C2 sweep timing, FP64 and FP32 (no e2e/cpu/ttt); prints one summary line each.
OUT=${1:-gpurun_out/qp}
mkdir -p "$OUT"
shift
for dt in f64 f32; do
  timeout 300 python bench.py --dtype $dt --steps 10 --warmup 3 --no-e2e --no-cpu --no-ttt "$@" > "$OUT/$dt.json" 2> "$OUT/$dt.err"
  python - "$OUT/$dt.json" "$dt" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1])); k = d["kernels"]
    print(sys.argv[2], "sweeps/s %.1f" % d["config"]["sweeps_per_s"], "fused ms %.3f" % (k["fused_sweep"]["ms_per_call"] or -1),
          "GB/s %.0f" % k["fused_sweep"].get("GB_per_s", 0), "h_apply ms %.3f" % k["h_apply"]["ms_per_call"], "clk", d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done
