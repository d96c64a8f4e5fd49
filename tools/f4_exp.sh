for m in 0 1 2 4 8 15; do
  if [ $m = 0 ]; then L=""; else L="build_ab/exp$m.so"; fi
  BICADMM_LIB_PATH=$L timeout 120 python bench.py --dtype f64 --steps 5 --warmup 2 --no-e2e --no-cpu --no-ttt > gpurun_out/e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e.json'));print('f64 R1 exp$m fused %.3f ms'%d['kernels']['fused_sweep']['ms_per_call'])" 2>/dev/null || echo "f64 exp$m failed"
  if [ $m = 0 ]; then L=""; else L="build_ab/exp${m}r2.so"; fi
  BICADMM_LIB_PATH=$L timeout 120 python bench.py --dtype f32 --steps 5 --warmup 2 --no-e2e --no-cpu --no-ttt > gpurun_out/e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e.json'));print('f32 R2 exp$m fused %.3f ms'%d['kernels']['fused_sweep']['ms_per_call'])" 2>/dev/null || echo "f32 exp$m failed"
done
