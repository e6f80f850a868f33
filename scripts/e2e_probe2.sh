# e2e leg (HostLayerPipeline): ramp schedules, alternating, bench.py only
mkdir -p gpurun_out; rm -f gpurun_out/e2e_*.txt
for r in 1 2 3; do
for c in 1,3,4,4,3,1 1,2,4,4,4,1 1,2,3,4,4,2 1,2,4,4,3,2; do
  timeout -s KILL 200 python bench.py --steps 5 --warmup 3 --no-cpu --no-dense --e2e-chunk $c 2>/dev/null | tail -1 >> gpurun_out/e2e_$c.txt
done; done
