#!/bin/bash
# One bench line per BASELINE.json config shape that fits one GPU (round-2 table).
OUT=${1:-gpurun_out/configs}
mkdir -p "$OUT"
timeout 300 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu > "$OUT/C1.json" 2> "$OUT/C1.err"
timeout 600 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu --no-ttt > "$OUT/C2.json" 2> "$OUT/C2.err"
timeout 600 python bench.py --config C2 --dtype f32 --steps 20 --warmup 5 --no-cpu --no-ttt > "$OUT/C2f32.json" 2> "$OUT/C2f32.err"
timeout 600 python bench.py --config C2ls --steps 20 --warmup 5 --no-cpu --no-ttt > "$OUT/C2ls.json" 2> "$OUT/C2ls.err"
timeout 900 python bench.py --config C4 --steps 4 --warmup 3 > "$OUT/C4.json" 2> "$OUT/C4.err"
timeout 900 python bench.py --config C3w --steps 4 --warmup 3 > "$OUT/C3w.json" 2> "$OUT/C3w.err"
timeout 900 python bench.py --config C3s --steps 4 --warmup 3 > "$OUT/C3s.json" 2> "$OUT/C3s.err"
timeout 900 python bench.py --config C5s --steps 4 --warmup 3 > "$OUT/C5s.json" 2> "$OUT/C5s.err"
timeout 900 python bench.py --config C5s --dtype f32 --steps 4 --warmup 3 > "$OUT/C5sf32.json" 2> "$OUT/C5sf32.err"
echo done
