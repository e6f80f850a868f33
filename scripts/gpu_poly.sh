mkdir -p gpurun_out; rm -f gpurun_out/ab2_poly*.txt
BSA_TC_EXP_POLY=3 timeout -s KILL 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -3 > gpurun_out/t_poly3.log
for r in 1 2; do for p in ${POLYS:-2 3 4}; do
  BSA_TC_EXP_POLY=$p timeout -s KILL 200 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 >> gpurun_out/ab2_poly$p.txt
done; done
