# N=1000 single-GPU leg (config 5's per-rank workload): kernel time + DRAM traffic
mkdir -p gpurun_out
timeout -s KILL 600 python bench.py --frames 1000 --steps 2 --warmup 1 --no-cpu --no-e2e --no-dense $BENCH_ARGS > gpurun_out/n1000_bench.json 2> gpurun_out/n1000_bench.err
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,sm__cycles_elapsed.avg.per_second \
  --clock-control none -k regex:bsa_tc_kernel -c 1 --csv python scripts/profile_step.py --frames 1000 --steps 1 $PROFILE_ARGS > gpurun_out/n1000_ncu.csv 2> gpurun_out/n1000_ncu.err
