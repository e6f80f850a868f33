# ncu evidence for the current build: launch list of one bench step and a
# --set full capture of the attention kernel and of the scoring kernels.
mkdir -p gpurun_out
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py --steps 1 > gpurun_out/ncu1.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:bsa_tc_kernel -s 2 -c 1 -o gpurun_out/prof_tc python scripts/profile_step.py --steps 1 > gpurun_out/ncu2.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"softsel|scores|pool" -s 4 -c 4 -o gpurun_out/prof_score python scripts/profile_step.py --steps 1 > gpurun_out/ncu3.log 2>&1
