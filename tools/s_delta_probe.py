"""How much the contact vertex set S changes between consecutive iterations of a C4 sequence
on the C3 mesh (decides whether updating Sigma_s = K_s^-1 by low-rank steps could replace the
full sweep): per iteration |S|, |added|, |removed|.  Usage: python tools/s_delta_probe.py [j] [frames]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import scenes  # noqa: E402
from paper_2312_02999_b200 import pd_ipc as P  # noqa: E402

j = int(sys.argv[1]) if len(sys.argv) > 1 else 0
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 32
sc = scenes.face_c3()
act = scenes.c4_actuation(sc, j)
s = P.Solver(sc, A=act(0)[None])
P.set_debug(s.h, 1)
prev = None
rows = []
for f in range(frames):
    for it in range(20):
        s.step(A_next=act(f)[None] if it == 0 else None, n_iters=1)
        _, _, S = P.get_contacts(s.h)
        cur = set(S.tolist())
        if prev is not None and (cur or prev):
            rows.append((f, it, len(cur), len(cur - prev), len(prev - cur)))
        prev = cur
s.close()
a = np.array([r[2:] for r in rows if r[2] > 0])
print(f"sequence {j}: {len(a)} iterations with contact; |S| mean {a[:, 0].mean():.0f}")
d = a[:, 1] + a[:, 2]
for q in (0, 50, 75, 90, 99, 100):
    print(f"  |added| + |removed| percentile {q}: {np.percentile(d, q):.0f}")
print("  fraction unchanged:", float(np.mean(d == 0)))
print("  last frames:", [r for r in rows[-25:]])
