# BASELINE.json configs beyond the headline bench line, one JSON line each
# into gpurun_out/configs/.  (config 1 = parity tests; config 3 N>1 and
# config 5 at 8 GPUs need torchrun on an 8-GPU box: see DESIGN.md.)
mkdir -p gpurun_out/configs
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
timeout -s KILL 300 python scripts/bench_config1.py > gpurun_out/configs/c1_n8.json 2>&1
# config 2: N=100 density sweep vs dense (tau = 0: exact density 1 - rho)
for rho in 0.0 0.5 0.6 0.7 0.75 0.8 0.9; do
  timeout -s KILL 300 $B --frames 100 --rho $rho > gpurun_out/configs/c2_rho$rho.json 2>&1
done
timeout -s KILL 300 $B --frames 100 --tau 0.4 --rho 0.8 > gpurun_out/configs/c2_t0.4_r0.8.json 2>&1
# config 4: pi3-shaped N=300 (4 register tokens, no camera token)
timeout -s KILL 400 $B --frames 300 --specials 4 > gpurun_out/configs/c4_pi3_n300.json 2>&1
# config 5 (single-GPU leg): N=1000, sparsity sweep
for rho in 0.5 0.75 0.9; do
  timeout -s KILL 900 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-dense --frames 1000 --rho $rho > gpurun_out/configs/c5_n1000_rho$rho.json 2>&1
done
# config 3: 24-layer stack at N=200, sparse vs dense
timeout -s KILL 900 python scripts/bench_stack.py --frames 200 --dense --fused --reps 1 > gpurun_out/configs/c3_stack_n200.json 2>&1
