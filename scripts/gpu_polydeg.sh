mkdir -p gpurun_out; rm -f gpurun_out/ab2_*.txt
BSA_LIB_VARIANT=d2 timeout -s KILL 300 python -m pytest tests/test_gpu_attention.py tests/test_gpu_shard.py tests/test_gpu_pipeline.py -x -q 2>&1 | tail -3 > gpurun_out/t_d2.log
for r in 1 2; do for v in d2 d3; do for p in 2 3 4; do
  BSA_LIB_VARIANT=$v BSA_TC_EXP_POLY=$p timeout -s KILL 200 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 >> gpurun_out/ab2_${v}p$p.txt
done; done; done
