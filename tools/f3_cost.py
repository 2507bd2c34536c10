"""Cost of the SURVEY 8(f) f3 options on C3 (BASELINE configs[2]): warm-started frame 30, 20
iterations, ms per iteration and the line-search stage with the default surrogate line search,
the true-energy line search (ls_energy = 1: one polar decomposition per tet and trial alpha), and
adaptive kappa (kappa_adapt_eps = d_hat).  Usage: python tools/f3_cost.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenes  # noqa: E402
from paper_2312_02999_b200 import pd_ipc as P  # noqa: E402

sc = scenes.face_c3()
for name, kw in (("default", {}), ("true_energy_ls", dict(ls_energy="true")),
                 ("adaptive_kappa", dict(kappa_adapt_eps=sc.d_hat))):
    s = P.Solver(sc, A=sc.actuation(29)[None], **kw)
    s.step(n_iters=20)
    s.step(A_next=sc.actuation(30)[None], n_iters=0)
    P.set_timing(s.h, True)
    P.kernel_times(s.h, reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    st = s.step(n_iters=20)[0]
    e1.record()
    torch.cuda.synchronize()
    kt = P.kernel_times(s.h, reset=True)
    s.close()
    print(json.dumps({"option": name, "ms_per_iter": e0.elapsed_time(e1) / 20, "kappa_last": st["kappa"],
                      "alpha_last": st["alpha"], "ls_trials_last": st["ls_trials"], "n_S_last": st["n_S"],
                      "line_search_ms_per_iter": round(kt.get("line_search", (0, 0))[0] / 20, 3)}), flush=True)
