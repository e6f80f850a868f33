# e2e leg: token-reordering copies (default) vs plain copies + pack pass, alternating
mkdir -p gpurun_out; rm -f gpurun_out/e2e3_*.txt
timeout -s KILL 400 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2 > gpurun_out/t_pipe.log
for r in 1 2 3; do
  timeout -s KILL 200 python bench.py --steps 5 --warmup 3 --no-cpu --no-dense 2>/dev/null | tail -1 >> gpurun_out/e2e3_part.txt
  timeout -s KILL 200 python bench.py --steps 5 --warmup 3 --no-cpu --no-dense --e2e-interleaved 2>/dev/null | tail -1 >> gpurun_out/e2e3_inter.txt
done
