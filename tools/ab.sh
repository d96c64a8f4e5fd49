#!/bin/bash
# A/B timing of two builds on the same box (interleaved):  tools/ab.sh <libA.so> <libB.so> <bench args...>
A=$1; B=$2; shift 2
for i in 1 2 3; do
  for L in "$A" "$B"; do
    BICADMM_LIB_PATH=$L timeout 400 python bench.py "$@" --steps ${AB_STEPS:-5} --warmup 3 --no-cpu --no-e2e --no-ttt > gpurun_out/ab.json 2>gpurun_out/ab.err
    python -c "
import json,sys
d=json.loads(open('gpurun_out/ab.json').read()); print('$L'.split('/')[-1], round(d['value'],1), round(d['ms_per_step'],3), {k:round(v['ms_per_call'],4) for k,v in d['kernels'].items() if v['launches']})
" || tail -3 gpurun_out/ab.err
  done
done
