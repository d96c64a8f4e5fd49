#!/bin/bash
# k_fused4 row-batch / axpy-delay study at configs[1] (FP64, FP32) and the Table-1 width.
for dt in f32 f64; do for R in 1 2 4; do for D in 1 2 3; do
  BICADMM_F4_R=$R BICADMM_F4_D=$D timeout 120 python bench.py --dtype $dt --steps 5 --warmup 2 --no-e2e --no-cpu --no-ttt "$@" > gpurun_out/rs.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/rs.json'));k=d['kernels']['fused_sweep'];print('$dt R=$R D=$D fused %.3f ms %.0f GB/s'%(k['ms_per_call'],k['GB_per_s']))" 2>/dev/null || echo "$dt R=$R D=$D n/a"
done; done; done
