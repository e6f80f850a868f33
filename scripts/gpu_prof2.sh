set -x
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_score.py tests/test_gpu_attention.py -x -q 2>&1 | tail -15 > gpurun_out/t_all.log
timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench200.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 12 --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py --steps 1 > gpurun_out/ncu1.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:bsa_tc_kernel -s 1 -c 1 -o gpurun_out/prof_tc python scripts/profile_step.py --steps 1 > gpurun_out/ncu2.log 2>&1
ls -la gpurun_out
