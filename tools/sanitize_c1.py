"""Small C1 run for compute-sanitizer (memcheck / racecheck / synccheck): 2 iterations of the
slabs scene in contact from the oracle-free GPU path, plus a 2-sequence lockstep step and the
gather backend.  Usage: compute-sanitizer --tool <tool> python tools/sanitize_c1.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import scenes  # noqa: E402
from paper_2312_02999_b200 import pd_ipc as P  # noqa: E402

sc = scenes.slabs_c1()
s = P.Solver(sc)
st = s.step(n_iters=6)[0]
print("C1 panel backend:", st["n_active"], st["n_S"], st["alpha"], flush=True)
s.close()
A = sc.actuation(0)
A2 = A.copy()
A2[:, 8] = 1.2
s = P.Solver(sc, A=np.stack([A, A2]), n_seq=2, reduced_backend=2)
st = s.step(n_iters=6)
print("C1 lockstep x2, gather backend:", [t["n_S"] for t in st], flush=True)
s.close()
