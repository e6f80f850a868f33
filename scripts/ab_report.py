import json, subprocess, sys
for v in sys.argv[1:]:
    try:
        d = json.loads(open(f'gpurun_out/ab_{v}.json').read().strip().splitlines()[-1])
        print(f"{v}: step {d['ms_per_step']:.2f} ms  kernel {d['stages_ms']['attention_kernel']:.2f} ms  "
              f"frac {d['roofline']['frac']:.3f}  clk {d['clocks']['sm_mhz']}")
    except Exception as e:
        print(v, 'ERR', e, open(f'gpurun_out/ab_{v}.err').read()[-500:])
    subprocess.run([sys.executable, 'scripts/trace_analyze.py', f'gpurun_out/trace_{v}.bin'])
