#!/bin/bash
# A/B of env settings on one box: /tmp/abenv.sh "ENV1" "ENV2" <bench args>
A=$1; B=$2; shift 2
for i in 1 2 3; do
  for E in "$A" "$B"; do
    env $E timeout 400 python bench.py "$@" --steps ${AB_STEPS:-5} --warmup 3 --no-cpu --no-e2e --no-ttt > gpurun_out/ab.json 2>gpurun_out/ab.err
    python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read()); print('$E', round(d['value'],1), {k:round(v['ms_per_call'],4) for k,v in d['kernels'].items() if v['launches']})
" || tail -3 gpurun_out/ab.err
  done
done
