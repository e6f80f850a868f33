# fused QKV projection: parity tests + timing of kernel variants (scripts/build_variants.sh)
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_qkv.py -x -q 2>&1 | tail -30 > gpurun_out/t_qkv.log
timeout -s KILL 300 python scripts/bench_qkv.py --layer > gpurun_out/bench_qkv.json 2> gpurun_out/bench_qkv.err
for v in ${QKV_VARIANTS:-}; do
  BSA_LIB_VARIANT=$v timeout -s KILL 200 python scripts/bench_qkv.py > gpurun_out/bench_qkv_$v.json 2>> gpurun_out/bench_qkv.err
done
