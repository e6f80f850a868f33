mkdir -p gpurun_out
BSA_TC_TRACE=gpurun_out/trace200.bin timeout -s KILL 200 python scripts/profile_step.py --steps 1 > gpurun_out/trace.log 2>&1
timeout -s KILL 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -3 > gpurun_out/t_attn.log
timeout -s KILL 200 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-dense > gpurun_out/bench_nt.json 2>&1
