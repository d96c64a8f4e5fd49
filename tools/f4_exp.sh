#!/bin/bash
# What bounds the single pass: timing variants of k_fused4 (BIC_F4_EXP bits: 1 skip the FMA
# blocks, 2 skip the prox, 4 skip the q wait; results are wrong by design) at configs[1].
#   for m in 1 2 4 6; do tools/build_f4_variant.sh exp$m -DBIC_F4_EXP=$m; done; tools/f4_exp.sh
for dt in f64 f32; do for m in 0 1 2 4 6; do
  if [ $m = 0 ]; then L=""; else L="build_ab/exp$m.so"; fi
  BICADMM_LIB_PATH=$L timeout 200 python bench.py --dtype $dt --steps 5 --warmup 3 --no-e2e --no-cpu --no-ttt > gpurun_out/e.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/e.json').read().strip().splitlines()[-1]);print('$dt exp$m fused %.3f ms'%d['kernels']['fused_sweep']['ms_per_call'])" 2>/dev/null || echo "$dt exp$m failed"
done; done
