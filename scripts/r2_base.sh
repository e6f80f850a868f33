set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,power.limit,clocks.max.sm --format=csv > gpurun_out/r2_gpu.txt
timeout -s KILL 600 python bench.py --no-cpu > gpurun_out/r2_bench0.json 2> gpurun_out/r2_bench0.err
bash scripts/gpu_sanitize.sh
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r2_tgpu.log
