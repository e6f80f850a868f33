mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_score.py tests/test_gpu_shard.py -x -q 2>&1 | tail -3 > gpurun_out/t_score.log
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:pool -c 4 --csv --log-file gpurun_out/pool.csv python scripts/profile_step.py --steps 1 > /dev/null 2>&1
