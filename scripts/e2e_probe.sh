# e2e leg (HostLayerPipeline) for several head-chunk schedules, bench.py only
mkdir -p gpurun_out; rm -f gpurun_out/e2e_*.txt
for r in 1 2; do
for c in 2 1,3,3,3,3,2,1 1,2,2,2,2,2,2,2,1 1,3,4,4,3,1 4; do
  timeout -s KILL 200 python bench.py --steps 5 --warmup 3 --no-cpu --no-dense --e2e-chunk $c 2>/dev/null | tail -1 >> gpurun_out/e2e_$c.txt
done; done
