export SPECS="base:2 l2h:2" TESTV=l2h
bash scripts/gpu_ab3.sh
for v in base l2h; do
BSA_LIB_VARIANT=$v timeout -s KILL 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:bsa_tc_kernel -s 2 -c 1 --csv python scripts/profile_step.py --steps 1 > gpurun_out/ncu_l2_$v.csv 2>&1
done
