set -u
mkdir -p gpurun_out
for R in 1 2 4 8; do
  for P in 0 1; do
    BICADMM_GEMV_R=$R BICADMM_GEMV_PERSISTENT=$P timeout 120 python tools/microbench.py >> gpurun_out/mb1.jsonl 2>>gpurun_out/mb1.err
  done
done
BICADMM_GEMV_R=4 timeout 120 python tools/microbench.py --dtype f32 >> gpurun_out/mb1.jsonl 2>>gpurun_out/mb1.err
cat gpurun_out/mb1.jsonl
