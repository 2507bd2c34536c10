"""GPU parity of reduced_backend 4, the paper's literal prescribed-region solve (PAPER.md:161-198,
Eq. 6-8; SURVEY 8(f) f1 "square"): the Schur complement of H-hat onto the whole W-supported
region R (S = R every iteration, Sigma_R computed once) must give the full solve's dx, like
every other backend.  Element by element against the oracle (which refactorises the full sparse
H-hat), in lockstep: g-hat to 1e-10, dx to 1e-8, alpha_m / alpha to 1e-10,
x to 1e-9 x bbox (tests/test_gpu_parity.py's tolerances).  The contact set C is compared bit for
bit; S is R by construction (checked), not the oracle's contact vertex set.
"""
import numpy as np
import pytest

import scenes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2312_02999_b200 import pd_ipc
    return pd_ipc


def _rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("scene", ["c1", "face_small"])
def test_region_backend_lockstep(P, scene):
    from oracle import OracleSolver, build_mesh
    if scene == "c1":
        sc = scenes.slabs_c1()
        A, n = sc.actuation(0), 10
    else:
        sc = scenes.face_small(n_frames=2)
        A = np.tile(np.eye(3).reshape(1, 9), (sc.n_tets, 1))
        A[:, 4] += 0.5 * sc.meta["lip_mask"]
        n = 6
    o = OracleSolver(sc)
    m = build_mesh(sc)
    R = np.unique(m.W.tocoo().col)
    R = R[m.free_pos[R] >= 0]                       # W-supported free vertices
    s = P.Solver(sc, A=A[None], reduced_backend=4)
    assert P.get_info(s.h)["reduced_backend"] == 4
    P.set_debug(s.h, 1)
    x = sc.rest.copy()
    for k in range(n):
        ref = o.iterate(x, A)
        P.set_positions(s.h, x)
        st = s.step(n_iters=1)[0]
        pt, ee, S = P.get_contacts(s.h)
        assert pt.shape[0] == ref["n_pt"] and ee.shape[0] == ref["n_ee"]
        assert np.array_equal(np.sort(S), np.sort(R)), k
        g = P.get_vector(s.h, sc.n_verts, 0)
        gref = np.zeros((sc.n_verts, 3))
        gref[o.mesh.free] = ref["ghat"].reshape(-1, 3)
        assert _rel(g, gref) < 1e-10, (k, _rel(g, gref))
        dx = P.get_vector(s.h, sc.n_verts, 1)
        assert _rel(dx, ref["dx"]) < 1e-8, (k, _rel(dx, ref["dx"]))
        assert abs(st["alpha_max"] - ref["alpha_m"]) <= 1e-10 * ref["alpha_m"]
        assert abs(st["alpha"] - ref["alpha"]) <= 1e-10 * ref["alpha_m"]
        assert np.abs(s.positions() - ref["x"]).max() < 1e-9 * sc.bbox_diag()
        x = ref["x"]
    s.close()


def test_region_backend_batch_equals_single(P):
    """Two lockstep sequences with S = R (batched Schur: both systems in one launch) are bit-identical
    to one sequence run alone, with the true-energy line search and adaptive kappa switched on too
    (every f-row option composed with the batched path)."""
    sc = scenes.slabs_c1()
    A = sc.actuation(0)
    kw = dict(reduced_backend=4, ls_energy="true", kappa_adapt_eps=sc.d_hat)
    one = P.Solver(sc, A=A[None], **kw)
    two = P.Solver(sc, A=np.stack([A, A]), n_seq=2, **kw)
    st1 = one.step(n_iters=12)[0]
    st2 = two.step(n_iters=12)
    for q in range(2):
        assert np.array_equal(two.positions(q), one.positions())
        assert st2[q]["kappa"] == st1["kappa"] and st2[q]["alpha"] == st1["alpha"]
    one.close()
    two.close()
