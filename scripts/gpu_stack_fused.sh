# compute-sanitizer (incl. proj_residual) + 24-layer stack sparse / fused / dense
mkdir -p gpurun_out/sanitize
rm -f gpurun_out/sanitize/summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 600 compute-sanitizer --tool $tool --print-limit 50 \
    python scripts/sanitize.py > gpurun_out/sanitize/$tool.log 2>&1
  echo "$tool rc=$? $(tail -1 gpurun_out/sanitize/$tool.log)" >> gpurun_out/sanitize/summary.txt
done
timeout -s KILL 1200 python scripts/bench_stack.py --frames 200 --fused --dense --reps 1 > gpurun_out/bench_stack.json 2> gpurun_out/bench_stack.err
timeout -s KILL 300 python scripts/bench_qkv.py > gpurun_out/bench_qkv.json 2>> gpurun_out/bench_stack.err
