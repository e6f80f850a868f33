# Quick iteration: attention parity + bench variants of the tensor-core kernel.
set -x
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -5 > gpurun_out/t_attn.log
for v in ${VARIANTS:-0}; do
  BSA_TC_EXP_POLY=$v timeout -s KILL 200 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-dense > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
done
tail -3 gpurun_out/t_attn.log
