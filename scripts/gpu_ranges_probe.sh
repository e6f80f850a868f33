python scripts/ranges_probe.py 200 1,2,3 > gpurun_out/ranges_probe.txt 2>&1
for n in 1 2; do
timeout -s KILL 600 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:bsa_tc_kernel -s 1 -c 1 --csv python scripts/ranges_probe.py 200 $n > gpurun_out/ncu_ranges_$n.csv 2>&1
done
