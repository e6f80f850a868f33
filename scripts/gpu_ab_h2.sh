# A/B: bf16 P (base lib, exp poly 2) vs fp16 P with HFMA2 polynomial exponentials (h2 lib)
mkdir -p gpurun_out; rm -f gpurun_out/abh_*.txt
for P in 2 4 6; do
BSA_LIB_VARIANT=h2 BSA_TC_F16P=1 BSA_TC_EXP_POLY=$P timeout -s KILL 400 python -m pytest tests/test_gpu_attention.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2 > gpurun_out/t_h2_p$P.log
done
for r in 1 2; do
for spec in base:0:2 h2:1:2 h2:1:3 h2:1:4 h2:1:5 h2:1:6 base:0:2; do
  IFS=: read v f p <<< "$spec"
  BSA_LIB_VARIANT=$v BSA_TC_F16P=$f BSA_TC_EXP_POLY=$p timeout -s KILL 200 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 >> gpurun_out/abh_${v}_f${f}_p$p.txt
done; done
