# A/B the library variants in csrc/build/<name>/: bench each (and trace each).
mkdir -p gpurun_out
for v in ${VARIANTS}; do
  BSA_LIB_VARIANT=$v timeout -s KILL 200 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-dense > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  BSA_LIB_VARIANT=$v BSA_TC_TRACE=gpurun_out/trace_$v.bin timeout -s KILL 200 python scripts/profile_step.py --steps 1 > /dev/null 2>&1
done
if [ -n "$TESTV" ]; then BSA_LIB_VARIANT=$TESTV timeout -s KILL 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -3 > gpurun_out/t_attn_$TESTV.log; fi
