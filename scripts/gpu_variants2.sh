mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -3 > gpurun_out/t_attn.log
for v in 0 1 2 3; do
  BSA_TC_EXP_POLY=$v timeout -s KILL 200 python bench.py --steps 4 --warmup 2 --no-cpu --no-e2e --no-dense > gpurun_out/var2_$v.json 2>&1
done
