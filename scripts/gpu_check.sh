set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 400 python -m pytest tests/test_gpu_score.py -x -q 2>&1 | tail -25 > gpurun_out/t_score.log
timeout -s KILL 400 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | tail -40 > gpurun_out/t_attn.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout -s KILL 300 python bench.py --frames 8 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench8.log 2>&1
timeout -s KILL 400 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench200.log 2>&1
tail -5 gpurun_out/*.log
