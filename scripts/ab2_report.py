import json, sys
for v in sys.argv[1:]:
    rows = [json.loads(l) for l in open(f'gpurun_out/ab2_{v}.txt') if l.startswith('{')]
    ks = [r['stages_ms']['attention_kernel'] for r in rows]
    cl = [r['clocks']['sm_mhz'] for r in rows]
    print(v, 'kernel ms', [round(k, 2) for k in ks], 'clk', cl, 'frac', [round(r['roofline']['frac'], 3) for r in rows])
