import sys, numpy as np
sys.path.insert(0, "/root/repo")
import scenes
from paper_2312_02999_b200 import pd_ipc as P
sc = scenes.face_c2()
s = P.Solver(sc)
for f in range(20):
    s.step(A_next=sc.actuation(f)[None], n_iters=20)
P.set_debug(s.h, 1)
same = tot = 0
prev = None
for f in range(20, 30):
    A = sc.actuation(f)[None]
    for it in range(20):
        st = s.step(A_next=A if it == 0 else None, n_iters=1)[0]
        _, _, S = P.get_contacts(s.h)
        if prev is not None and S.shape == prev.shape and np.array_equal(S, prev):
            same += 1
        tot += 1
        prev = S
print("iterations", tot, "S unchanged from previous", same)
