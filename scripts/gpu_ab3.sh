# A/B over (library variant, exp-poly split) pairs: SPECS="name:poly name:poly ..."
mkdir -p gpurun_out
if [ -n "$TESTV" ]; then BSA_LIB_VARIANT=$TESTV timeout -s KILL 400 python -m pytest tests/test_gpu_attention.py tests/test_gpu_shard.py -x -q 2>&1 | tail -3 > gpurun_out/t_ab.log; fi
rm -f gpurun_out/ab2_*.txt
for r in 1 2; do
for spec in ${SPECS}; do
  v="${spec%%:*}"; p="${spec#*:}"
  BSA_LIB_VARIANT=$v BSA_TC_EXP_POLY=$p timeout -s KILL 200 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-dense $BENCH_ARGS 2>/dev/null | tail -1 >> gpurun_out/ab2_${v}_p$p.txt
done; done
