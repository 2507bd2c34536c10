"""O0: one-time setup of the oracle (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

PAPER.md:72-85 (section 2.1, Eq. 1-2): F_i(x) = G_i x, w_i = rest volume, H = sum_i w_i G_i^T G_i.
PAPER.md:143 (section 3.1): embedded surface s = W x.
SURVEY.md 8(c) O0 fixes the readings used here:
  D_m = [X1-X0, X2-X0, X3-X0], det D_m > 0, w = det/6, B = D_m^{-1};
  g_c = row c-1 of B (c = 1..3), g_0 = -(g_1+g_2+g_3);  F = sum_c x_c g_c^T;
  L_uv = sum_i w_i g_{i,u} . g_{i,v}  with H = L (x) I3 (vertex-major xyz DOFs);
  surface edges = unique sorted vertex pairs of the surface triangles;
  W_{j,v} = embed_w[j][c] for v = corner c of embed_tet[j] (exact zeros dropped).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp


@dataclass
class OracleMesh:
    n: int
    tets: np.ndarray          # (T,4)
    w: np.ndarray             # (T,) rest volumes
    B: np.ndarray             # (T,3,3) D_m^{-1}
    g: np.ndarray             # (T,4,3) corner gradients g_{i,c}
    Lap: sp.csr_matrix        # (n,n) scalar PD matrix, H = Lap (x) I3
    fixed: np.ndarray         # sorted Dirichlet ids
    free: np.ndarray          # sorted free ids
    free_pos: np.ndarray      # (n,) index of vertex in `free`, -1 for fixed
    tris: np.ndarray          # (N_t,3) surface-vertex ids
    edges: np.ndarray         # (N_e,2) sorted unique surface edges
    W: sp.csr_matrix          # (N_s, n)
    rest: np.ndarray          # (n,3)

    @property
    def n_free(self) -> int:
        return int(self.free.size)

    def deformation_gradients(self, x: np.ndarray) -> np.ndarray:
        """F_i = sum_c x_{v_c} g_{i,c}^T  (Eq. 1)."""
        Xc = x[self.tets]                                    # (T,4,3)
        return np.einsum("tca,tcb->tab", Xc, self.g)

    def H_dense_free(self) -> np.ndarray:
        """Dense H = L (x) I3 on free DOFs (small fixtures only)."""
        Lff = self.Lap[self.free][:, self.free].toarray()
        return np.kron(Lff, np.eye(3))


def _surface_edges(tris: np.ndarray) -> np.ndarray:
    if tris.shape[0] == 0:
        return np.zeros((0, 2), dtype=np.int64)
    e = np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]])
    e = np.sort(e, axis=1)
    return np.unique(e, axis=0)


def build_mesh(scene) -> OracleMesh:
    """O0; validates the rest mesh like pd_ipc_create does."""
    X = np.asarray(scene.rest, dtype=np.float64)
    tets = np.asarray(scene.tets, dtype=np.int64)
    n = X.shape[0]
    if tets.size and (tets.min() < 0 or tets.max() >= n):
        raise ValueError("tet index out of range")
    Xt = X[tets]
    Dm = np.stack([Xt[:, 1] - Xt[:, 0], Xt[:, 2] - Xt[:, 0], Xt[:, 3] - Xt[:, 0]], axis=2)
    det = np.linalg.det(Dm)
    if not (det > 0).all():
        raise ValueError("inverted or degenerate rest tet (det D_m <= 0)")
    w = det / 6.0
    B = np.linalg.inv(Dm)
    g = np.empty((tets.shape[0], 4, 3))
    g[:, 1:, :] = B                                          # row c-1 of B
    g[:, 0, :] = -(B[:, 0, :] + B[:, 1, :] + B[:, 2, :])
    # L_uv = sum_i w_i g_{i,u} . g_{i,v}  (Eq. 2 with H = L (x) I3)
    T = tets.shape[0]
    rows, cols, vals = [], [], []
    for u in range(4):
        for v in range(4):
            rows.append(tets[:, u])
            cols.append(tets[:, v])
            vals.append(w * np.einsum("ta,ta->t", g[:, u], g[:, v]))
    Lap = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                        shape=(n, n)).tocsr()
    fixed = np.unique(np.asarray(scene.fixed, dtype=np.int64))
    if fixed.size == 0:
        raise ValueError("no Dirichlet vertices: H is singular (SPEC.md:78)")
    is_fixed = np.zeros(n, bool)
    is_fixed[fixed] = True
    free = np.nonzero(~is_fixed)[0]
    free_pos = -np.ones(n, dtype=np.int64)
    free_pos[free] = np.arange(free.size)
    tris = np.asarray(scene.surf_tris, dtype=np.int64).reshape(-1, 3)
    et = np.asarray(scene.embed_tet, dtype=np.int64)
    ew = np.asarray(scene.embed_w, dtype=np.float64).reshape(-1, 4)
    Ns = et.size
    if Ns:
        if (ew < 0).any() or (ew > 1).any() or (np.abs(ew.sum(1) - 1.0) > 1e-12).any():
            raise ValueError("W row not convex")
    wr, wc, wv = [], [], []
    for c in range(4):
        nz = ew[:, c] != 0.0
        wr.append(np.nonzero(nz)[0])
        wc.append(tets[et[nz], c])
        wv.append(ew[nz, c])
    W = sp.coo_matrix((np.concatenate(wv) if Ns else np.zeros(0),
                       (np.concatenate(wr) if Ns else np.zeros(0, int),
                        np.concatenate(wc) if Ns else np.zeros(0, int))),
                      shape=(Ns, n)).tocsr()
    return OracleMesh(n=n, tets=tets, w=w, B=B, g=g, Lap=Lap, fixed=fixed, free=free,
                      free_pos=free_pos, tris=tris, edges=_surface_edges(tris), W=W, rest=X)
