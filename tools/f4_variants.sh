#!/bin/bash
# time the single-pass sweep of A/B library variants: tools/f4_variants.sh name1 name2 ... (build_ab/<name>.so; "base" = in-tree)
for v in "$@"; do
  for dt in f64 f32; do
    L=build_ab/$v.so; [ "$v" = base ] && L=""
    if [ -n "$L" ] && [ "$dt" = f32 ] && [ -f build_ab/${v}r2.so ]; then L=build_ab/${v}r2.so; fi
    BICADMM_LIB_PATH=$L timeout 120 python bench.py --dtype $dt --steps 5 --warmup 2 --no-e2e --no-cpu --no-ttt > gpurun_out/v.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/v.json'));k=d['kernels']['fused_sweep'];print('$v $dt fused %.3f ms %.0f GB/s'%(k['ms_per_call'],k['GB_per_s']))" 2>/dev/null || echo "$v $dt n/a"
  done
done
