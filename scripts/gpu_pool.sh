# pool8 variants: parity (score tests) and ncu device time of the two pools
mkdir -p gpurun_out
BSA_LIB_VARIANT=${TESTV:-} timeout -s KILL 300 python -m pytest tests/test_gpu_score.py -x -q 2>&1 | tail -3 > gpurun_out/t_score.log
for v in ${VARIANTS}; do
BSA_LIB_VARIANT=$v timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pool8 -c 4 --csv --log-file gpurun_out/pool_$v.csv python scripts/profile_step.py --steps 1 > /dev/null 2>&1
done
