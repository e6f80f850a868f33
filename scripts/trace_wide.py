"""Summarise a BSA_TC_TRACE dump of the one-CTA-per-SM kernel (CTA 0).

Events per key tile (BSA_TR in bsa_attn_tc.cu): 0 K TMA issued, 1 S MMAs
issued, 2 PV MMAs issued, 3 K tile arrived (MMA warp passed KFULL), 4 the
owning group's quarter-0 warp starts waiting for S, 8 S ready (SFULL
passed), 12 exps done, 16 P published."""
import sys

import numpy as np

NE, NT = 20, 512
t = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/trace200.bin',
                dtype=np.uint64).reshape(NE, NT).astype(np.int64)
ev = [0, 1, 2, 3, 4, 8, 12, 16]
ok = (t[ev] > 0).all(axis=0)
v = t[:, ok][:, 50:]
v = v - v[ev].min()
med = lambda x: float(np.median(x))
print('tiles', v.shape[1], ' tile period (P publish)', med(np.diff(v[16])),
      ' S-issue period', med(np.diff(v[1])), ' PV-issue period', med(np.diff(v[2])))
print('softmax: wait for S', med(v[8] - v[4]), ' S ready -> exps done', med(v[12] - v[8]),
      ' exps done -> P published', med(v[16] - v[12]))
print('group: P published(j) -> starts waiting for S(j+4)', med(v[4][4:] - v[16][:-4]))
print('P published -> PV issued', med(v[2] - v[16]))
print('S issued -> S ready (softmax saw it)', med(v[8] - v[1]))
print('S issued before the group started waiting for it', med(v[4] - v[1]))
print('K TMA issued -> K arrived', med(v[3] - v[0]), ' K arrived -> S issued', med(v[1] - v[3]))
for q in (10, 50, 90):
    print(f'p{q}: wait S {np.percentile(v[8]-v[4], q):.0f}  exps {np.percentile(v[12]-v[8], q):.0f}  '
          f'P->PV {np.percentile(v[2]-v[16], q):.0f}')
# producer / MMA-warp detail: 9 producer chose K(j) (about to wait KEMPTY),
# 6 producer passed VEMPTY for V(j), 11 MMA warp starts waiting KFULL(j),
# 10 MMA warp starts PV(j) (waits PFULL), 7 passed PFULL, 5 passed VFULL
if (t[[5, 6, 7, 9, 10, 11]] > 0).all(axis=0).sum() > 60:
    print('producer: K(j) chosen -> K TMA issued', med(v[0] - v[9]), '  V(j) TMA issued', med(v[6] - v[0]))
    print('MMA: start wait KFULL(j) -> passed', med(v[3] - v[11]))
    print('MMA: PV(j) start -> PFULL passed', med(v[7] - v[10]), ' -> VFULL passed', med(v[5] - v[7]),
          ' -> PV issued', med(v[2] - v[5]))
    print('V(j) TMA issued -> VFULL passed', med(v[5] - v[6]))
if (t[13] > 0).sum() > 60:
    nb = 6
    print(f'S warp: KFULL passed -> PFREE passed {med(v[13] - v[3]):.0f};  PV(j-{nb}) issued -> PFREE seen by S(j) {med(v[13][nb:] - v[2][:-nb]):.0f}')
    print(f'S(j) issue vs P(j-{nb}) published {med(v[1][nb:] - v[16][:-nb]):.0f};  S(j) issued vs P(j-4) published {med(v[1][4:] - v[16][:-4]):.0f}')
    print('S warp loop: S(j) issued -> S(j+1) issued', med(np.diff(v[1])))
