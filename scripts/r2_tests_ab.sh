mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q --durations=10 2>&1 | tail -25 > gpurun_out/r2_tgpu_full.log
VARIANTS="${VARIANTS:-base}" RUNS=${RUNS:-2} bash scripts/gpu_ab_r2.sh
