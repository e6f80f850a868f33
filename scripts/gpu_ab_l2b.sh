mkdir -p gpurun_out; rm -f gpurun_out/ab2_*.txt
for r in 1 2 3; do
for spec in base:2 l2h:2 l2h:2 base:2; do
  v="${spec%%:*}"; p="${spec#*:}"
  BSA_LIB_VARIANT=$v BSA_TC_EXP_POLY=$p timeout -s KILL 200 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 >> gpurun_out/ab2_${v}_p$p.txt
done; done
