import sys, time
sys.path.insert(0, "/root/repo")
import torch, scenes
from paper_2312_02999_b200 import pd_ipc as P
sc = scenes.face_c2()
s = P.Solver(sc)
for f in range(20):
    s.step(A_next=sc.actuation(f)[None], n_iters=20)
for on in (False, True, False, True):
    P.set_timing(s.h, on)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for f in range(20, 26):
        s.step(A_next=sc.actuation(f)[None], n_iters=20)
    e1.record(); torch.cuda.synchronize()
    print("timing", on, "ms/iter", e0.elapsed_time(e1) / 120)
