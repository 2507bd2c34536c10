"""Runs C2 into the contact regime with PDIPC_TRACE set and analyses the forward-solve items of
the last traced iteration: span, per-item wait/work times, and the chain of supernodes that
finishes last (the critical path).  Usage: python tools/trace_c2.py [frames] [trace-file]"""
import os
import struct
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 22
path = sys.argv[2] if len(sys.argv) > 2 else "/tmp/pdipc_trace.bin"
os.environ["PDIPC_TRACE"] = path
os.environ["PDIPC_DUMP_SUPERNODES"] = path + ".sn"
import scenes  # noqa: E402
from paper_2312_02999_b200 import pd_ipc as P  # noqa: E402

sc = scenes.face_c2()
P.debug_factor_solve(sc)          # host factor only: writes the supernode dump
s = P.Solver(sc)
for f in range(frames):
    st = s.step(A_next=sc.actuation(f)[None], n_iters=20)
s.close()
print("last frame stats", {k: st[0][k] for k in ("n_cand", "n_active", "n_S")})
raw = open(path, "rb").read()
recs, off = [], 0
while off < len(raw):
    (n,) = struct.unpack_from("i", raw, off)
    off += 4
    recs.append(np.frombuffer(raw, np.uint64, 4 * n, off).reshape(n, 4).astype(np.int64))
    off += 32 * n
print("traced iterations", len(recs))
sn = np.loadtxt(path + ".sn", dtype=np.int64)
w, nr, par = sn[:, 2], sn[:, 3], sn[:, 4]
nonempty = [r for r in recs if len(r)]
if nonempty:
    tr = nonempty[-1]
    t0 = tr[:, 1].min()
    sid, tk = tr[:, 0] >> 16, tr[:, 0] & 0xFFFF
    disp, ready, done = tr[:, 1] - t0, tr[:, 2] - t0, tr[:, 3] - t0
    work = done - ready
    print(f"items {len(tr)}  span {done.max() / 1e3:.1f} us  work mean {work.mean() / 1e3:.2f} us  "
          f"p50 {np.median(work) / 1e3:.2f}  p90 {np.percentile(work, 90) / 1e3:.2f}  max {work.max() / 1e3:.2f}")
    print(f"sum of work {work.sum() / 1e3:.0f} us over {len(tr)} items")
    # per supernode: finish time = max done over its items
    fin = np.zeros(len(w), np.int64)
    start = np.full(len(w), 1 << 62, np.int64)
    for i in range(len(tr)):
        fin[sid[i]] = max(fin[sid[i]], done[i])
        start[sid[i]] = min(start[sid[i]], ready[i])
    # walk from the last-finishing root down the latest-finishing child
    r = int(np.argmax(fin))
    chain = [r]
    while True:
        ch = np.nonzero(par == chain[-1])[0]
        if len(ch) == 0:
            break
        chain.append(int(ch[np.argmax(fin[ch])]))
    print("critical chain (root first): s, w, nr, items, ready-after-children us, work span us")
    for c in chain:
        ch = np.nonzero(par == c)[0]
        cf = fin[ch].max() if len(ch) else 0
        its = np.nonzero(sid == c)[0]
        print(f"  {c:4d} w {w[c]:3d} nr {nr[c]:4d} items {len(its):3d}  wait {(start[c] - cf) / 1e3:6.2f}  "
              f"span {(fin[c] - start[c]) / 1e3:6.2f}  maxwork {work[its].max() / 1e3:6.2f}")


# ---- fused Schur kernel: time between consecutive grid barriers (last traced call)
sp = path + ".schur"
if os.path.exists(sp):
    raw = open(sp, "rb").read()
    rec = 4 + 8 * 1024
    nrec = len(raw) // rec
    (nS,) = struct.unpack_from("i", raw, (nrec - 1) * rec)
    for r in range(max(0, nrec - 6), nrec):
        (nS,) = struct.unpack_from("i", raw, r * rec)
        ts = np.frombuffer(raw, np.uint64, 1024, r * rec + 4).astype(np.int64)
        ts = ts[ts > 0]
        d = np.diff(ts) / 1e3
        print(f"schur nS {nS}: {len(d)} barrier intervals, total {d.sum():.1f} us")
        print("  intervals (us):", " ".join(f"{x:.1f}" for x in d))
