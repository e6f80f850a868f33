# Round-2 full pass: quick check, GPU parity suite, smoke, driver-shaped bench
# (20 steps), ragged/LPT bench lines, N=1000 leg, ncu launch list and --set
# full captures of the attention and scoring kernels.
O=${O:-gpurun_out/r2full}; mkdir -p $O

timeout -s KILL 90 python scripts/quick_check.py > $O/quick.log 2>&1 || { echo "quick check failed" >> $O/quick.log; exit 1; }
timeout -s KILL 1500 python -m pytest tests -m gpu -q --durations=10 2>&1 | tail -30 > $O/t_gpu.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
timeout -s KILL 300 python bench.py --mask ragged --no-cpu --no-e2e --no-dense > $O/bench_ragged_lpt.json 2> $O/bench_ragged_lpt.err
timeout -s KILL 300 python bench.py --mask ragged --schedule natural --no-cpu --no-e2e --no-dense > $O/bench_ragged_natural.json 2> $O/bench_ragged_natural.err
timeout -s KILL 300 python bench.py --schedule natural --no-cpu --no-e2e --no-dense > $O/bench_uniform_natural.json 2> $O/bench_uniform_natural.err
timeout -s KILL 600 python bench.py --frames 1000 --steps 2 --warmup 1 --no-cpu --no-e2e --no-dense > $O/bench_n1000.json 2> $O/bench_n1000.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python scripts/profile_step.py --steps 1 > $O/ncu1.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:bsa_tc_kernel -s 2 -c 1 -o $O/prof_tc python scripts/profile_step.py --steps 1 > $O/ncu2.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"softsel|scores|pool" -s 4 -c 4 -o $O/prof_score python scripts/profile_step.py --steps 1 > $O/ncu3.log 2>&1
