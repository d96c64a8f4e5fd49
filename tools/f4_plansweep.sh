#!/bin/bash
# k_fused4 launch-plan study (row batch R, row groups GR, axpy delay D) on one bench preset:
#   tools/f4_plansweep.sh <tag> <bench args...>      e.g.  tools/f4_plansweep.sh c5s --config C5s --nodes 2
# Infeasible plans fall back to the auto plan (the line then repeats the auto plan's time).
TAG=$1; shift
mkdir -p gpurun_out/plans
for R in 1 2 4; do for G in 1 2 3 4 6; do for D in 1 2; do
  BICADMM_F4_R=$R BICADMM_F4_GROUPS=$G BICADMM_F4_D=$D timeout 200 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-ttt "$@" > gpurun_out/plans/$TAG.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/plans/$TAG.json').read().strip().splitlines()[-1]);k=d['kernels']['fused_sweep'];print('$TAG R=$R G=$G D=$D fused %.3f ms %.0f GB/s'%(k['ms_per_call'],k['GB_per_s']))" 2>/dev/null || echo "$TAG R=$R G=$G D=$D n/a"
done; done; done
timeout 200 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-ttt "$@" > gpurun_out/plans/$TAG.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/plans/$TAG.json').read().strip().splitlines()[-1]);k=d['kernels']['fused_sweep'];print('$TAG auto fused %.3f ms %.0f GB/s'%(k['ms_per_call'],k['GB_per_s']))"
