"""Summarise tools/_bin/attn_trace output: per-phase clocks of the ping-pong kernel."""
import sys
import numpy as np

rows = [l.strip().split(',') for l in open(sys.argv[1]) if l[:1].isdigit()]
hdr = [l for l in open(sys.argv[1]) if l.startswith('#')]
A = {}
for r in rows:
    A.setdefault(int(r[0]), []).append([int(x) for x in r[1:]])
A = {k: np.array(v) for k, v in A.items()}
sl = slice(20, min(150, len(A[0]) - 2))
print(hdr[0].strip() if hdr else '')
m = A[0]
print("MMA period %.0f" % np.diff(m[sl, 1]).mean(),
      " ".join("%s %.0f" % (n, (m[sl, i + 1] - m[sl, i]).mean()) for i, n in
               enumerate(['vfull', 'S_A', 'PV_A', 'S_B', 'PV_B'], 1)))
for nm, k in (('A', 1), ('B', 2)):
    x = A[k]
    s2 = slice(sl.start + 1, sl.stop + 1)
    print("%s period %.0f  sfull-wait %.0f pass1 %.0f pvwait %.0f pass2 %.0f tail %.0f" % (
        nm, np.diff(x[sl, 1]).mean(), (x[s2, 1] - x[sl, 5]).mean(), (x[sl, 2] - x[sl, 1]).mean(),
        (x[sl, 3] - x[sl, 2]).mean(), (x[sl, 4] - x[sl, 3]).mean(), (x[sl, 5] - x[sl, 4]).mean()))
