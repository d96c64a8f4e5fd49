# C4 (softmax, 80 GB) kernel-variant sweep: rows per GEMV-C task x rows in flight in GEMV-T-C
set -u
mkdir -p gpurun_out
for R in 1 2 4; do for U in 1 2 4; do
  BICADMM_GEMVC_R=$R BICADMM_GTC_U=$U timeout 300 python bench.py --config C4 --steps 2 --warmup 2 --no-e2e > gpurun_out/c4_${R}_${U}.json 2>gpurun_out/c4_${R}_${U}.err
  python -c "
import json,sys
d=json.loads(open('gpurun_out/c4_${R}_${U}.json').read()); k=d['kernels']
print('R=$R U=$U', round(d['value'],3), 'gemv', round(k['gemv']['ms_per_launch'],2), 'gemv_t', round(k['gemv_t_partial']['ms_per_launch'],2))" || tail -3 gpurun_out/c4_${R}_${U}.err
done; done
