"""Runs C2 frames into the contact regime with PDIPC_TRACE set; analyses forward-solve items."""
import os, sys, struct
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scenes
from paper_2312_02999_b200 import pd_ipc as P
sc = scenes.face_c2()
s = P.Solver(sc)
P.set_timing(s.h, True)
for f in range(0, 26):
    st = s.step(A_next=sc.actuation(f)[None], n_iters=20)
    if f % 5 == 0:
        print(f, "cand", st[0]["n_cand"], "active", st[0]["n_active"], "nS", st[0]["n_S"], {k: round(v[0] / max(v[1], 1), 3) for k, v in P.kernel_times(s.h, reset=True).items()}, flush=True)
s.close()
