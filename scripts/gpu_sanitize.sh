# compute-sanitizer over every kernel family (scripts/sanitize.py, small shapes).
mkdir -p gpurun_out/sanitize
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 420 compute-sanitizer --tool $tool --print-limit 50 \
    python scripts/sanitize.py > gpurun_out/sanitize/$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize/summary.txt
done
