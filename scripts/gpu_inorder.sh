mkdir -p gpurun_out; rm -f gpurun_out/ab2_*.txt gpurun_out/t_inord*.log
for r in 1 2 3; do BSA_LIB_VARIANT=inord timeout -s KILL 400 python -m pytest tests/test_gpu_attention.py tests/test_gpu_shard.py tests/test_gpu_acceptance.py tests/test_gpu_pipeline.py -x -q 2>&1 | tail -2 >> gpurun_out/t_inord.log; done
for r in 1 2; do for v in inord cur; do
  BSA_LIB_VARIANT=$v timeout -s KILL 200 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 >> gpurun_out/ab2_$v.txt
done; done
