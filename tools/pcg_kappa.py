"""f2: the paper's PCG baseline vs the direct reduced solves, and its kappa x 10 experiment
("If we increase its initial value by 10x, the cost of the conjugate gradient solver
would nearly double ... our method is a direct solver ... independent of kappa").  Per scene and
kappa: a warm-started frame (20 iterations from rest under the frame-(F-1) actuation, then 20
timed iterations at frame F); G-step ms per iteration (Table 1's column) and CG iterations.
Usage: python tools/pcg_kappa.py [scenes...]  (default C2 C3)"""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenes  # noqa: E402
from paper_2312_02999_b200 import pd_ipc as P  # noqa: E402


def run(sc, frame, backend, iters=20):
    s = P.Solver(sc, A=sc.actuation(frame - 1)[None], reduced_backend=backend, cg_tol=1e-10)
    s.step(n_iters=20)
    s.step(A_next=sc.actuation(frame)[None], n_iters=0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = s.step(n_iters=iters)[0]
    e1.record()
    torch.cuda.synchronize()
    info = P.get_info(s.h)
    s.close()
    return {"backend": {1: "panel", 2: "gather", 3: "pcg"}[info["reduced_backend"]],
            "ms_per_iter": e0.elapsed_time(e1) / iters, "gstep_ms_per_iter": st["ms"]["gstep"] / iters,
            "cg_iters_per_newton_iter": st["cg_iters"] / iters, "n_S_last": st["n_S"]}


names = sys.argv[1:] or ["C2", "C3"]
for name in names:
    base = {"C2": scenes.face_c2, "C3": scenes.face_c3}[name]()
    for kf in (1.0, 10.0):
        sc = dataclasses.replace(base, kappa=base.kappa * kf)
        for be in ((1, 3) if name == "C2" else (2, 3)):
            r = run(sc, 30, be)
            r.update({"scene": name, "kappa_factor": kf})
            print(json.dumps(r), flush=True)
