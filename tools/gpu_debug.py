"""Step-by-step GPU check of C1 against the oracle with verbose prints (debug aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scenes
from oracle import OracleSolver
from paper_2312_02999_b200 import pd_ipc as P

print(P.build_info(), flush=True)
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
sc = {"c1": scenes.slabs_c1, "box": lambda: scenes.box_c5("10k"), "small": scenes.face_small}[name]()
o = OracleSolver(sc)
t = time.time()
s = P.Solver(sc)
print("create ok %.2fs" % (time.time() - t), flush=True)
P.set_debug(s.h, 1)
x = sc.rest.copy()
A = sc.actuation(0)
for k in range(int(sys.argv[2]) if len(sys.argv) > 2 else 6):
    ref = o.iterate(x, A)
    P.set_positions(s.h, x)
    st = s.step(n_iters=1)[0]
    pt, ee, S = P.get_contacts(s.h)
    g = P.get_vector(s.h, sc.n_verts, 0)
    dx = P.get_vector(s.h, sc.n_verts, 1)
    gref = np.zeros((sc.n_verts, 3)); gref[o.mesh.free] = ref["ghat"].reshape(-1, 3)
    xg = s.positions()
    print(f"it {k}: nC gpu {pt.shape[0]}+{ee.shape[0]} ref {ref['n_pt']}+{ref['n_ee']} | nS {S.size} ref {ref['S'].size} "
          f"eqS {np.array_equal(S, ref['S'])} | g rel {np.abs(g-gref).max()/max(np.abs(gref).max(),1e-300):.2e} "
          f"| dx rel {np.abs(dx-ref['dx']).max()/max(np.abs(ref['dx']).max(),1e-300):.2e} | am {st['alpha_max']:.6f}/{ref['alpha_m']:.6f} "
          f"a {st['alpha']:.6f}/{ref['alpha']:.6f} | x err {np.abs(xg-ref['x']).max():.2e} | ms {st['ms']['total']:.2f}", flush=True)
    x = ref["x"]
s.close()
print("done", flush=True)
