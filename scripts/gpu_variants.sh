mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -3 > gpurun_out/t_attn.log
BSA_TC_F16P=1 BSA_TC_EXP_POLY=0 timeout -s KILL 300 python -m pytest tests/test_gpu_attention.py -x -q -k tc 2>&1 | tail -3 > gpurun_out/t_attn_f16.log
for v in "0 0" "1 0" "2 0" "3 0" "4 0" "0 1" "2 1"; do
  set -- $v
  BSA_TC_EXP_POLY=$1 BSA_TC_F16P=$2 timeout -s KILL 200 python bench.py --steps 4 --warmup 2 --no-cpu --no-e2e --no-dense > gpurun_out/var_$1_$2.json 2>&1
done
