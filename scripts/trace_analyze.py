import sys
import numpy as np
NE = 20
t = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/trace200.bin', dtype=np.uint64).reshape(NE, 512).astype(np.int64)
base = t[t > 0].min()
t = np.where(t > 0, t - base, -1)
keep = [0, 1, 2] + list(range(4, 20))
v = t[:, (t[keep].min(axis=0) >= 0)][:, 50:]
med = lambda x: float(np.median(x))
W, G, E, P = 4, 8, 12, 16
print('tiles', v.shape[1], ' tile period (warp0)', med(np.diff(v[P])))
for w in range(4):
    print(f'warp {w}: wait S {med(v[G+w]-v[W+w]):7.0f}  ld S->exp done {med(v[E+w]-v[G+w]):7.0f}  '
          f'exp done->bar passed {med(v[P+w]-v[E+w]):6.0f}  bar->next wait {med(v[W+w][1:]-v[P+w][:-1]):6.0f}')
print('warp0: bar passed -> PV issued', med(v[2] - v[P]))
print('S issue lead (warp0 got S(j) - S issued(j)) [same SMSP as mma? no]', med(v[G] - v[1]))
