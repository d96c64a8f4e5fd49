#!/bin/bash
# single pass (--sweep 2) vs two passes (--sweep 1) per sweep at narrow widths (auto-choice crossover)
for dt in f64 f32; do for n in 500 800 1000 1400 2000 3000; do
  m=$((60000000 / n))
  for sw in 1 2; do
    timeout 200 python bench.py --dtype $dt --n $n --m $m --nodes 4 --loss logistic --kappa 20 --sweep $sw --steps 5 --warmup 2 --no-e2e --no-cpu --no-ttt > gpurun_out/x.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/x.json'));print('$dt n=$n sweep=$sw sweeps/s %.1f'%d['config']['sweeps_per_s'])" 2>/dev/null || echo "$dt n=$n sweep=$sw n/a"
  done
done; done
