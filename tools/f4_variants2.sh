#!/bin/bash
# A/B the single-pass sweep on narrow rows: tools/f4_variants2.sh variant...  (Table-1 width, C5 block width)
for v in "$@"; do
  L=build_ab/$v.so; [ "$v" = base ] && L=""
  for shape in "4 75000 4000 ls" "4 60000 6250 hinge" "4 150000 2000 logistic"; do
    set -- $shape
    for dt in f64 f32; do
      BICADMM_LIB_PATH=$L timeout 120 python bench.py --dtype $dt --nodes $1 --m $2 --n $3 --loss $4 --kappa 100 --steps 5 --warmup 2 --no-e2e --no-cpu --no-ttt > gpurun_out/v2.json 2>/dev/null
      python -c "import json;d=json.load(open('gpurun_out/v2.json'));k=d['kernels']['fused_sweep'];print('$v n=$3 $dt fused %.3f ms %.0f GB/s'%(k['ms_per_call'],k['GB_per_s']))" 2>/dev/null || echo "$v n=$3 $dt n/a"
    done
  done
done
