"""C4 probe (BASELINE.json configs[3]): B sequences of the C3 mesh in one lockstep handle.
Prep: every sequence from rest with its frame-(F-1) actuation for `prep` iterations, then
timed lockstep iterations at frame F.  Usage: python tools/c4_probe.py [B] [prep] [iters] [F]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import scenes  # noqa: E402
from paper_2312_02999_b200 import pd_ipc as P  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
prep = int(sys.argv[2]) if len(sys.argv) > 2 else 20
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 5
F = int(sys.argv[4]) if len(sys.argv) > 4 else 30
t0 = time.time()
sc = scenes.face_c3()
acts = [scenes.c4_actuation(sc, j) for j in range(B)]
A0 = np.stack([a(F - 1) for a in acts])
A1 = np.stack([a(F) for a in acts])
print("gen_s", round(time.time() - t0, 1), flush=True)
t0 = time.time()
s = P.Solver(sc, A=A0, n_seq=B)
print("create_s", round(time.time() - t0, 1), "mem_GB", round(torch.cuda.mem_get_info()[1] / 1e9 - torch.cuda.mem_get_info()[0] / 1e9, 1), flush=True)
t0 = time.time()
st = s.step(n_iters=prep)
torch.cuda.synchronize()
print("prep_s", round(time.time() - t0, 1), "n_S", [x["n_S"] for x in st][:8], "mean", np.mean([x["n_S"] for x in st]), flush=True)
A1d = torch.from_numpy(A1).cuda()
s.step(A_next=A1, n_iters=0)
P.set_timing(s.h, True)
P.kernel_times(s.h, reset=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
st = s.step(n_iters=iters)
e1.record()
torch.cuda.synchronize()
kt = P.kernel_times(s.h, reset=True)
ms = e0.elapsed_time(e1)
print(json.dumps({"B": B, "ms_per_lockstep_iter": ms / iters, "ms_per_seq_iter": ms / iters / B,
                  "n_S_mean": float(np.mean([x["n_S"] for x in st])), "n_S_max": int(max(x["n_S"] for x in st)),
                  "reused": [x["sigma_reused"] for x in st][:8],
                  "alpha": [x["alpha"] for x in st][:8],
                  "stage_ms_total_per_iter": {k: round(v[0] / iters, 3) for k, v in kt.items() if v[1]},
                  "stage_ms_per_launch": {k: round(v[0] / v[1], 3) for k, v in kt.items() if v[1]},
                  "seq_ms": {k: round(float(np.mean([x["ms"][k] for x in st])) / iters, 3) for k in ("ipc", "gstep", "ccd", "ls", "misc", "total")}}), flush=True)
s.close()
