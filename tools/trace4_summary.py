"""Summarise tools/_bin/attn_trace output for the Q/P-in-TMEM kernel (vc_attn_tc4.cu)."""
import sys
import numpy as np

rows = [l.strip().split(',') for l in open(sys.argv[1]) if l[:1].isdigit()]
print([l.strip() for l in open(sys.argv[1]) if l.startswith('#')][0])
A = {}
for r in rows:
    A.setdefault(int(r[0]), []).append([int(x) for x in r[2:]])
A = {k: np.array(v) for k, v in A.items()}
m = A[0]
j = np.arange(20, min(150, len(m) - 2))
names = ['vfull', 'PV_A', 'kfull', 'S_A', 'PV_B', 'S_B']
print("MMA period %.0f | " % np.diff(m[j, 0]).mean() +
      " ".join("%s %.0f" % (names[i], (m[j, i] - m[j, i - 1]).mean()) for i in range(1, 6)) +
      " wrap %.0f" % (m[j + 1, 0] - m[j, 5]).mean())
for sw in range(16):
    if sw not in A.__class__.keys(A) and (1 + sw) not in A:
        continue
    x = A[1 + sw]
    print("warp %2d: sfull-wait %4.0f ld+max+xchg %4.0f rescale %4.0f exp+st %4.0f tail %4.0f" % (
        2 + sw, (x[j + 1, 0] - x[j, 4]).mean(), (x[j, 1] - x[j, 0]).mean(), (x[j, 2] - x[j, 1]).mean(),
        (x[j, 3] - x[j, 2]).mean(), (x[j, 4] - x[j, 3]).mean()))
if len(sys.argv) > 2:
    a, b = A[1], A[9]
    base = a[40, 0]
    ev = []
    for jj in range(40, 42):
        for i, n in enumerate(names):
            ev.append((m[jj, i] - base, 'MMA', jj, n))
        for nm, x in (('A', a), ('B', b)):
            for i, n in enumerate(['sfull', 'xchg', 'rescale', 'exp', 'pfull']):
                ev.append((x[jj, i] - base, nm, jj, n))
    for e in sorted(ev):
        print("%6d %-4s %3d %s" % e)
