"""f1 ablation: the reduced-solve backends (panel, precomputed-region gather, the paper's prescribed-region
solve with S = R) behind the same
dx contract, on C2 and C3 (BASELINE configs[1], [2]): warm-started frame, ms per iteration and
stage times.  Usage: python tools/backend_ablation.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import scenes  # noqa: E402
from paper_2312_02999_b200 import pd_ipc as P  # noqa: E402


def run(name, sc, frame, backend, prep=20, iters=20):
    s = P.Solver(sc, A=sc.actuation(frame - 1)[None], reduced_backend=backend)
    info = P.get_info(s.h)
    s.step(n_iters=prep)
    s.step(A_next=sc.actuation(frame)[None], n_iters=0)
    P.set_timing(s.h, True)
    P.kernel_times(s.h, reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    st = s.step(n_iters=iters)[0]
    e1.record()
    torch.cuda.synchronize()
    kt = P.kernel_times(s.h, reset=True)
    x = s.positions()
    s.close()
    return {"scene": name, "backend": {1: "panel", 2: "gather", 4: "region"}[info["reduced_backend"]],
            "region_size": info["region_size"], "ms_per_iter": e0.elapsed_time(e1) / iters,
            "n_S_last": st["n_S"], "sigma_reused": st["sigma_reused"],
            "stage_ms_per_iter": {k: round(v[0] / iters, 3) for k, v in kt.items() if v[1]}}, x


for name, mk, frame in (("C2", scenes.face_c2, 30), ("C3", scenes.face_c3, 30)):
    sc = mk()
    xs = []
    for be in (1, 2, 4):
        r, x = run(name, sc, frame, be)
        xs.append(x)
        print(json.dumps(r), flush=True)
    print(json.dumps({"scene": name, "max_position_difference_between_backends":
                      float(max(np.abs(xs[0] - y).max() for y in xs[1:])),
                      "bbox_diag": sc.bbox_diag()}), flush=True)
