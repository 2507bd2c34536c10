"""Runs the C2 sequence into the contact regime, then one frame inside an NVTX range 'timed'
(for `ncu --nvtx --nvtx-include timed/`).  Prints per-group device times of that frame."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import scenes
from paper_2312_02999_b200 import pd_ipc as P
start = int(sys.argv[1]) if len(sys.argv) > 1 else 25
sc = scenes.face_c2()
s = P.Solver(sc)
for f in range(start):
    s.step(A_next=sc.actuation(f)[None], n_iters=20)
P.set_timing(s.h, True)
P.kernel_times(s.h, reset=True)
torch.cuda.nvtx.range_push("timed")
st = s.step(A_next=sc.actuation(start)[None], n_iters=20)
torch.cuda.nvtx.range_pop()
kt = P.kernel_times(s.h, reset=True)
print("frame", start, "stats", {k: st[0][k] for k in ("n_cand", "n_active", "n_S", "alpha")})
print({k: round(v[0] / max(v[1], 1), 4) for k, v in kt.items() if v[1]})
s.close()
