"""Phase breakdown of the dense Schur kernel (PDIPC_TRACE): runs C3 into contact with the
trace on and prints, per traced iteration, n_c and the microseconds of P0 (y_S, K = V^T V),
P1 (Sigma_s = K^-1), P2 (assembly), P3 (Cholesky), P4 (back substitution), P5 (t, Z).
Usage: python tools/schur_phases.py [frames]"""
import os
import struct
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
path = os.path.join(tempfile.mkdtemp(), "tr.bin")
os.environ["PDIPC_TRACE"] = path
import numpy as np  # noqa: E402

import scenes  # noqa: E402
from paper_2312_02999_b200 import pd_ipc as P  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 24
sc = scenes.face_c3()
s = P.Solver(sc)
for f in range(frames):
    s.step(A_next=sc.actuation(f)[None], n_iters=20 if f < frames - 1 else 4)
s.close()
data = open(path + ".schur", "rb").read()
rec = 4 + 8 * 1024
rows = []
for i in range(len(data) // rec):
    nS = struct.unpack_from("i", data, i * rec)[0]
    pr = np.frombuffer(data, dtype=np.uint64, count=1024, offset=i * rec + 4).astype(np.int64)
    mk = [0] + [int(pr[1000 + k]) for k in range(1, 6)]
    # end of P5: the stamp after the CTA-0 stamp of 'CTA 0 done with t = B u' (1007) when the
    # gather backend's end stamp (1006) is absent
    e6 = int(pr[1006]) if pr[1006] else int(pr[1007])
    ts = [pr[mk[k]] for k in range(6)] + [pr[e6]]
    rows.append((nS, [(ts[k + 1] - ts[k]) / 1e3 for k in range(6)], (pr[int(pr[1007])] - pr[mk[5]]) / 1e3))
    if pr[996] and pr[995]:
        print(f"  (n_c {nS}: P2 CTA 0 assembly rows {(pr[996] - pr[mk[2]]) / 1e3:.1f} us, b rows {(pr[995] - pr[996]) / 1e3:.1f} us)")
for nS, ph, tbu in rows[-12:]:
    print(f"n_c {nS:5d}  " + "  ".join(f"P{k} {v:8.1f}" for k, v in enumerate(ph)) +
          f"  total {sum(ph):8.1f} us  (t = B u: {tbu:.1f})")
# large-system P3 look-ahead detail of the last traced iteration: per panel iteration q, the
# panel group's time (its update of panel q + the panel factorisation) and the update group's
nS, _, _ = rows[-1]
i = len(data) // rec - 1
pr = np.frombuffer(data, dtype=np.uint64, count=1024, offset=i * rec + 4).astype(np.int64)
m3 = int(pr[1003])
print("P3 detail (us from the iteration start): q  npg  panel_upd_done  panel_done  update_done  end;  wu_coef", pr[997] / 1000)
for q in range(100):
    if pr[800 + q] == 0:
        break
    t0 = pr[m3 + q]
    t1 = pr[m3 + q + 1]
    print(q, int(pr[800 + q]), round((pr[500 + q] - t0) / 1e3, 1) if pr[500 + q] else "-",
          round((pr[600 + q] - t0) / 1e3, 1), round((pr[700 + q] - t0) / 1e3, 1) if pr[700 + q] else "-",
          round((t1 - t0) / 1e3, 1))
# per-column detail of panels 0 and 12: after the diagonal factor / TRSM / intra-panel update
# barriers (us from the panel-update-done stamp)
for qq, off in ((0, 900), (12, 940)):
    if pr[off] == 0:
        continue
    base = pr[500 + qq]
    cols = [[round(float(pr[off + 3 * c + j] - base) / 1e3, 1) for j in range(3)] for c in range(10) if pr[off + 3 * c]]
    print(f"panel {qq} columns (start, after TRSM, after update) us after its panel update:", cols)
# P1 sweep detail of the last traced iteration with S changed: per pivot step, phase A (U, the
# previous column) and phase B (rank-64 update + next pivot) in us, from the grid-barrier stamps
for i in range(len(data) // rec - 1, -1, -1):
    pr = np.frombuffer(data, dtype=np.uint64, count=1024, offset=i * rec + 4).astype(np.int64)
    m1, m2 = int(pr[1001]), int(pr[1002])
    if m2 - m1 > 8:
        st = [pr[j] for j in range(m1, m2 + 1)]
        d = np.diff(np.array(st, dtype=np.float64)) / 1e3
        A, B = d[1:-2:2], d[2:-2:2]
        print(f"P1 detail (n_c {struct.unpack_from('i', data, i * rec)[0]}): first pivot {d[0]:.1f} us, "
              f"phase A mean {A.mean():.1f} (first {A[:3].round(1).tolist()}), phase B mean {B.mean():.1f} "
              f"(first {B[:3].round(1).tolist()}, last {B[-3:].round(1).tolist()}), steps {len(B)}")
        break
