"""Embedding construction (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

PAPER.md:143 (section 3.1): the collision proxy is a surface embedded in the tet mesh, s = W x.
SPEC.md:53-61 (build_embedding) and :81 (tie rule) fix the construction: every surface point gets
the barycentric coordinates of the tet that contains it (within tolerance), a point on a face
shared by two tets going to the LOWER-index tet.  Written plainly: for every point, every tet in
index order, barycentric coordinates by numpy.linalg.solve of D_m lambda = p - X_0; the first tet
with all four coordinates >= -tol wins; coordinates clamped at 0 and renormalised.
"""
from __future__ import annotations

import numpy as np


def build_embedding(tets: np.ndarray, X: np.ndarray, points: np.ndarray, tol: float = 1e-9):
    """-> (embed_tet (P,), embed_w (P, 4)); ValueError for a point outside every tet."""
    tets = np.asarray(tets, dtype=np.int64)
    X = np.asarray(X, dtype=np.float64)
    points = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    Dm = np.stack([X[tets[:, 1]] - X[tets[:, 0]], X[tets[:, 2]] - X[tets[:, 0]],
                   X[tets[:, 3]] - X[tets[:, 0]]], axis=2)                     # (T, 3, 3)
    et = np.zeros(points.shape[0], dtype=np.int64)
    ew = np.zeros((points.shape[0], 4))
    for q, p in enumerate(points):
        lam = np.linalg.solve(Dm, (p - X[tets[:, 0]])[:, :, None])[:, :, 0]   # (T, 3)
        bary = np.concatenate([1.0 - lam.sum(axis=1, keepdims=True), lam], axis=1)
        inside = np.nonzero((bary >= -tol).all(axis=1))[0]
        if inside.size == 0:
            raise ValueError(f"point {q} lies outside every tet")
        t = int(inside[0])                                                    # lowest index
        w = np.maximum(bary[t], 0.0)
        et[q] = t
        ew[q] = w / w.sum()
    return et, ew
