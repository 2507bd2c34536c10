"""C5 pure-PD sweep (BASELINE.json configs[4]): per size, local-step and gather
HBM GB/s from the library's CUDA-event kernel timers, and pure-PD iterations/s.
Usage: python tools/c5_sweep.py [sizes...]   (default 10k 50k 100k 300k)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenes  # noqa: E402
from paper_2312_02999_b200 import pd_ipc as P  # noqa: E402


def run(size, iters=20, reps=3):
    sc = scenes.box_c5(size)
    t0 = time.time()
    s = P.Solver(sc)
    setup = time.time() - t0
    info = P.get_info(s.h)
    s.step(n_iters=2)                                   # warm-up
    P.set_timing(s.h, True)
    P.kernel_times(s.h, reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        s.step(n_iters=iters)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    kt = P.kernel_times(s.h, reset=True)
    s.close()
    T, n = sc.n_tets, sc.n_verts
    nf = n - len(sc.fixed)
    lb = T * (16 + 72 + 48 + 8 + 96) + n * 32         # local step algorithmic bytes
    gb = nf * (8 + 32) + 4 * T * (4 + 24)               # gather
    loc_us = kt["local_step"][0] / kt["local_step"][1] * 1e3
    gat_us = kt["gather"][0] / kt["gather"][1] * 1e3
    # triangular solves: the factor (nnz(L) doubles of Q blocks) read once per solve + the
    # right-hand side in and the solution out ([nf][4] doubles each)
    sb = info["nnz_L"] * 8 + nf * 32 * 2
    fw_us = kt["w_el_forward"][0] / kt["w_el_forward"][1] * 1e3
    bw_us = kt["backward_solve"][0] / kt["backward_solve"][1] * 1e3
    return {"size": size, "tets": T, "verts": n, "setup_s": round(setup, 1),
            "nnz_L": info["nnz_L"], "supernodes": info["supernodes"], "etree_depth": info["etree_depth"],
            "forward_solve_us": fw_us, "forward_solve_GBps": sb / fw_us / 1e3,
            "backward_solve_us": bw_us, "backward_solve_GBps": sb / bw_us / 1e3,
            "iters_per_s": reps * iters / (ms / 1e3),
            "local_step_us": loc_us, "local_step_GBps": lb / loc_us / 1e3,
            "gather_us": gat_us, "gather_GBps": gb / gat_us / 1e3,
            "stage_ms_per_iter": {k: v[0] / max(v[1], 1) for k, v in kt.items() if v[1]}}


if __name__ == "__main__":
    for size in (sys.argv[1:] or ["10k", "50k", "100k", "300k", "1M", "2M"]):
        print(json.dumps(run(size)), flush=True)
