mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:bsa_tc_kernel -s 1 -c 1 -o gpurun_out/prof_tc3 python scripts/profile_step.py --steps 1 > gpurun_out/ncu3.log 2>&1
