# fused QKV projection: compute-sanitizer (small shapes, all kernel families),
# ncu capture of the GEMM at N=200, 24-layer stack sparse vs fused.
mkdir -p gpurun_out/sanitize
rm -f gpurun_out/sanitize/summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 600 compute-sanitizer --tool $tool --print-limit 50 \
    python scripts/sanitize.py > gpurun_out/sanitize/$tool.log 2>&1
  echo "$tool rc=$? $(tail -1 gpurun_out/sanitize/$tool.log)" >> gpurun_out/sanitize/summary.txt
done
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:qkv_pool -s 3 -c 1 \
  -o gpurun_out/prof_qkv python scripts/bench_qkv.py --reps 2 > gpurun_out/ncu_qkv.log 2>&1
timeout -s KILL 900 python scripts/bench_stack.py --fused --reps 1 > gpurun_out/bench_stack.json 2> gpurun_out/bench_stack.err
