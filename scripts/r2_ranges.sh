mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_key_ranges.py tests/test_gpu_attention.py tests/test_gpu_shard.py tests/test_gpu_api_guards.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -15 > gpurun_out/t_ranges.log
timeout -s KILL 600 python bench.py --frames 1000 --steps 2 --warmup 1 --no-cpu --no-e2e --no-dense > gpurun_out/n1000_r_bench.json 2> gpurun_out/n1000_r_bench.err
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second \
  --clock-control none -k regex:bsa_tc_kernel -c 1 --csv python scripts/profile_step.py --frames 1000 --steps 1 > gpurun_out/n1000_r_ncu.csv 2> gpurun_out/n1000_r_ncu.err
timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-dense > gpurun_out/n200_r_bench.json 2> gpurun_out/n200_r_bench.err
timeout -s KILL 120 python bench.py --gpus 2 --steps 1 --warmup 0 > gpurun_out/gpus2.out 2> gpurun_out/gpus2.err; echo "gpus2 rc=$?" >> gpurun_out/gpus2.err
