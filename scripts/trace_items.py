"""Item transitions in a BSA_TC_TRACE dump of the one-CTA-per-SM kernel
(CTA 0, softmax warp 0): 14 item start (popped), 15 last tile published,
17 O complete (OFULL), 18 epilogue done.  Reports the per-item overhead."""
import sys

import numpy as np

t = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/trace200.bin',
                dtype=np.uint64).reshape(20, 512).astype(np.int64)
n = int(((t[14] > 0) & (t[18] > 0)).sum())
s, e15, e17, e18 = t[14][:n], t[15][:n], t[17][:n], t[18][:n]
med = lambda x: float(np.median(x))
print('items traced', n)
print('item duration (start -> epilogue done)', med(e18 - s))
print('last P published -> O complete', med(e17 - e15), ' epilogue', med(e18 - e17))
print('epilogue done -> next item start', med(s[1:] - e18[:-1]))
tot = e18[-1] - s[0]
busy = (e15 - s).sum()
print(f'fraction of CTA-0 time between items (after last P, before next tiles): {1 - busy / tot:.3%}')
