"""Summarise a BSA_TC_TRACE dump (clock64 per pipeline event of CTA 0).

Events (see bsa_attn_tc.cu BSA_TR): 0 producer K/V TMA issued, 1 S MMAs
issued, 2 PV MMAs issued, 3 K tile arrived (MMA passed KFULL), 4+w softmax
warp w starts waiting for S, 8+w S loaded to registers, 12+w exps done,
16+w P published (PFULL arrive)."""
import sys

import numpy as np

NE, NT = 20, 512
t = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/trace200.bin',
                dtype=np.uint64).reshape(NE, NT).astype(np.int64)
ok = (t > 0).all(axis=0)
v = t[:, ok][:, 50:]
base = v.min()
v = v - base
med = lambda x: float(np.median(x))
print('tiles', v.shape[1], ' tile period (warp0 P publish)', med(np.diff(v[16])))
for w in range(4):
    print(f'warp {w}: wait S {med(v[8+w]-v[4+w]):7.0f}  S loaded->exps done {med(v[12+w]-v[8+w]):7.0f}  '
          f'exps done->P published {med(v[16+w]-v[12+w]):6.0f}  publish->next wait {med(v[4+w][1:]-v[16+w][:-1]):6.0f}')
print('P published (last warp) -> PV issued', med(v[2] - v[16:20].max(axis=0)))
print('S issued -> S loaded (warp0)', med(v[8] - v[1]))
print('K/V TMA issued -> K arrived', med(v[3] - v[0]))
print('K arrived -> S issued', med(v[1] - v[3]))
print('S issued(j+1) - PV issued(j)', med(v[1][1:] - v[2][:-1]))
print('lead: S issued(j) before softmax starts waiting for it', med(v[4] - v[1]))
