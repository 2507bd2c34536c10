"""embedding construction (build_embedding).

Oracle pins (textbook special cases, SPEC's own examples): a point at a mesh vertex gets a unit
W row; a tet centroid gets (1/4, 1/4, 1/4, 1/4); random interior points are reproduced by W X to
1e-12; a point on a face shared by two tets goes to the lower-index tet; a point outside raises.
The library's host function (pd_ipc_build_embedding) must return the oracle's tets exactly and
its weights to 1e-12.  GPU: the surface export pd_ipc_surface_positions equals W x."""
import numpy as np
import pytest

import scenes
from oracle.embedding import build_embedding


def _two_tets():
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 1]], float)
    T = np.array([[0, 1, 2, 3], [1, 2, 3, 4]], np.int64)       # share face (1, 2, 3)
    return T, X


def test_oracle_embedding_special_cases():
    T, X = _two_tets()
    et, ew = build_embedding(T, X, X[[0, 4]])
    assert et.tolist() == [0, 1]
    assert np.array_equal(ew[0], [1, 0, 0, 0]) and np.array_equal(ew[1], [0, 0, 0, 1])
    c = X[T[1]].mean(0)
    et, ew = build_embedding(T, X, c[None])
    assert et[0] == 1 and np.abs(ew[0] - 0.25).max() < 1e-15
    f = X[[1, 2, 3]].mean(0)                                    # on the shared face
    et, ew = build_embedding(T, X, f[None])
    assert et[0] == 0                                           # lowest index
    assert np.abs(ew[0] @ X[T[0]] - f).max() < 1e-15
    with pytest.raises(ValueError):
        build_embedding(T, X, np.array([[2.0, 2.0, 2.0]]))


def test_oracle_embedding_reproduces_random_points():
    sc = scenes.face_small()
    rng = np.random.default_rng(8)
    t = rng.integers(0, sc.n_tets, 300)
    b = rng.dirichlet(np.ones(4), 300)
    pts = np.einsum("pc,pcd->pd", b, sc.rest[sc.tets[t]])
    et, ew = build_embedding(sc.tets, sc.rest, pts)
    rec = np.einsum("pc,pcd->pd", ew, sc.rest[sc.tets[et]])
    assert np.abs(rec - pts).max() < 1e-12 * np.abs(sc.rest).max()
    assert (et <= t).all()                                      # never a higher tet than one containing it


@pytest.fixture(scope="module")
def P():
    from paper_2312_02999_b200 import pd_ipc
    return pd_ipc


def test_library_embedding_matches_oracle(P):
    sc = scenes.face_small()
    rng = np.random.default_rng(9)
    t = rng.integers(0, sc.n_tets, 400)
    b = rng.dirichlet(np.ones(4), 400)
    pts = np.einsum("pc,pcd->pd", b, sc.rest[sc.tets[t]])
    pts = np.concatenate([pts, sc.rest[:50], sc.surface_rest()[:100]])   # vertices, faces, edges
    et, ew = build_embedding(sc.tets, sc.rest, pts)
    et2, ew2 = P.build_embedding(sc.tets, sc.rest, pts)
    assert np.array_equal(et2, et)
    assert np.abs(ew2 - ew).max() < 1e-12
    with pytest.raises(P.PdIpcError) as e:
        P.build_embedding(sc.tets, sc.rest, np.array([[1.0, 1.0, 1.0]]))
    assert e.value.code == P.E_MESH


@pytest.mark.gpu
def test_surface_export_matches_w_x(P):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import build_mesh
    sc = scenes.face_small(n_frames=2)
    s = P.Solver(sc)
    s.step(A_next=sc.actuation(1)[None], n_iters=5)
    x = s.positions()
    out = P.surface_positions(s.h, sc.n_surf_verts)
    ref = build_mesh(sc).W @ x
    assert np.abs(out - ref).max() <= 1e-14 * np.abs(ref).max()
    s.close()
