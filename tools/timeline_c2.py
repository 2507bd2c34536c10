"""Per-iteration timeline of the kernel groups (start/stop offsets in us from the local step's
start, CUDA events on both streams) for C2 frames in the contact regime.
Usage: PDIPC_TIMELINE=1 python tools/timeline_c2.py [start_frame] [frames]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PDIPC_TIMELINE", "1")
import scenes  # noqa: E402
from paper_2312_02999_b200 import pd_ipc as P  # noqa: E402

start = int(sys.argv[1]) if len(sys.argv) > 1 else 25
nfr = int(sys.argv[2]) if len(sys.argv) > 2 else 1
sc = scenes.face_c2()
s = P.Solver(sc)
os.environ["PDIPC_TIMELINE"] = "0"
for f in range(start):
    s.step(A_next=sc.actuation(f)[None], n_iters=20)
P.set_timing(s.h, True)
for f in range(start, start + nfr):
    st = s.step(A_next=sc.actuation(f)[None], n_iters=20)
    print("frame", f, {k: st[0][k] for k in ("n_cand", "n_active", "n_S", "alpha")}, flush=True)
kt = P.kernel_times(s.h, reset=True)
print({k: round(v[0] / max(v[1], 1) * 1e3, 1) for k, v in kt.items() if v[1]})
s.close()
