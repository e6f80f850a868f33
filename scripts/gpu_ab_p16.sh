# exp split at 1/16 granularity (p16 lib: POLY of every 16 pairs, spread) vs base (2 of 8)
mkdir -p gpurun_out; rm -f gpurun_out/ab2_*.txt
BSA_LIB_VARIANT=p16 BSA_TC_EXP_POLY=5 timeout -s KILL 400 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -2 > gpurun_out/t_p16.log
for r in 1 2 3; do
for spec in base:2 p16:3 p16:4 p16:5 p16:6; do
  v="${spec%%:*}"; p="${spec#*:}"
  if [ "$v" = base ]; then lib=""; else lib=$v; fi
  BSA_LIB_VARIANT=$lib BSA_TC_EXP_POLY=$p timeout -s KILL 200 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 >> gpurun_out/ab2_${v}_p$p.txt
done; done
