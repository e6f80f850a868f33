# Full GPU pass: parity tests, smoke, bench (with CPU baseline), reference arm,
# ncu launch list + full capture of the attention and scoring kernels.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/t_gpu.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout -s KILL 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py --steps 1 > gpurun_out/ncu1.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:bsa_tc_kernel -s 2 -c 1 -o gpurun_out/prof_tc python scripts/profile_step.py --steps 1 > gpurun_out/ncu2.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"softsel|scores|pool" -s 4 -c 4 -o gpurun_out/prof_score python scripts/profile_step.py --steps 1 > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out
