# compute-sanitizer over every kernel family (scripts/sanitize.py, small shapes);
# a second memcheck/racecheck pass with BSA_SCORESEL=0 covers the three-kernel
# scoring path.
mkdir -p gpurun_out/sanitize
rm -f gpurun_out/sanitize/summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 600 compute-sanitizer --tool $tool --print-limit 50 \
    python scripts/sanitize.py > gpurun_out/sanitize/$tool.log 2>&1
  echo "$tool rc=$? $(grep -c 'ERROR SUMMARY: 0 errors\|RACECHECK SUMMARY: 0 hazards' gpurun_out/sanitize/$tool.log) $(tail -1 gpurun_out/sanitize/$tool.log)" >> gpurun_out/sanitize/summary.txt
done
for tool in memcheck racecheck; do
  BSA_SCORESEL=0 timeout -s KILL 600 compute-sanitizer --tool $tool --print-limit 50 \
    python scripts/sanitize.py > gpurun_out/sanitize/${tool}_threekernel.log 2>&1
  echo "$tool (BSA_SCORESEL=0) rc=$? $(tail -1 gpurun_out/sanitize/${tool}_threekernel.log)" >> gpurun_out/sanitize/summary.txt
done
