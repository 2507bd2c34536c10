"""C3 probe (BASELINE.json configs[2]): run the 300k-tet two-slit face into contact and report
per-iteration time, n_c and stage times.  Usage: python tools/c3_probe.py [frames] [start]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenes  # noqa: E402
from paper_2312_02999_b200 import pd_ipc as P  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 60
t0 = time.time()
sc = scenes.face_c3()
s = P.Solver(sc)
print("setup_s", round(time.time() - t0, 1), "tets", sc.n_tets, "verts", sc.n_verts,
      "surface tris", sc.surf_tris.shape[0], flush=True)
for f in range(frames):
    P.set_timing(s.h, True)
    P.kernel_times(s.h, reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = s.step(A_next=sc.actuation(f)[None], n_iters=20)[0]
    e1.record()
    torch.cuda.synchronize()
    kt = P.kernel_times(s.h, reset=True)
    if f % 5 == 4 or st["n_S"] > 0:
        print(json.dumps({"frame": f, "ms_per_iter": e0.elapsed_time(e1) / 20, "n_S": st["n_S"],
                          "n_active": st["n_active"], "alpha": st["alpha"], "reused": st["sigma_reused"],
                          "stages": {k: round(v[0] / max(v[1], 1), 3) for k, v in kt.items() if v[1]}}),
              flush=True)
s.close()
