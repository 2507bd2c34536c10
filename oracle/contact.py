"""O3-O5 contact set, contact vertex set and pulled-back barrier derivatives
(TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

PAPER.md:88 (section 2.2): the constraint set C holds the primitive pairs (vertex-triangle,
edge-edge) whose distance is below d_0.  SURVEY.md 8(c) O3 / Z14 / Z16: enumerate ALL PT pairs
(j, f) with j not in f and ALL EE pairs (e, e') with e < e' sharing no vertex; C = pairs with
d^2 < d_hat^2 (d_hat*d_hat computed once); sorted lists (PT by (j, f), EE by (e, e')).
PAPER.md:143 (section 3.1): grad B = W^T grad_s B, and script-B = W^T hess_s B W.
PAPER.md:204-238 (section 3.2, Eq. 9-10) with SURVEY Z18: S = sorted unique free vertices with a
structurally nonzero W entry for any of the 4 surface vertices of any pair in C.

Enumeration is brute force.  For meshes too large for an all-pairs sweep a k-d tree
(scipy.spatial.cKDTree, a library neighbour search) first discards pairs whose bounding
spheres are farther apart than the margin; this is exact because the distance between two
primitives is at least the distance between their bounding spheres.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.spatial import cKDTree

from . import barrier as Bm
from . import distance as D

BRUTE_LIMIT = 20_000           # all-pairs sweep below this many pairs (tests force it)


def _pt_all(tris, Ns):
    j = np.repeat(np.arange(Ns), tris.shape[0])
    f = np.tile(np.arange(tris.shape[0]), Ns)
    return j, f


def _ee_all(Ne):
    e, e2 = np.triu_indices(Ne, k=1)
    return e, e2


def pt_candidates(s, tris, margin):
    """PT pairs (j, f), j not in f, that may lie within `margin`; sorted by (j, f)."""
    Ns, Nt = s.shape[0], tris.shape[0]
    if Ns * Nt <= BRUTE_LIMIT:
        j, f = _pt_all(tris, Ns)
    else:
        cen = (s[tris[:, 0]] + s[tris[:, 1]] + s[tris[:, 2]]) / 3.0
        rad = np.max(np.linalg.norm(s[tris] - cen[:, None, :], axis=2))
        tree = cKDTree(cen)
        lists = tree.query_ball_point(s, r=margin + rad * (1 + 1e-9) + 1e-300)
        j = np.repeat(np.arange(Ns), [len(l) for l in lists])
        f = np.concatenate([np.asarray(l, dtype=np.int64) for l in lists]) if Ns else np.zeros(0, int)
    inc = (tris[f] == j[:, None]).any(axis=1)
    j, f = j[~inc], f[~inc]
    o = np.lexsort((f, j))
    return j[o], f[o]


def ee_candidates(s, edges, margin):
    """EE pairs (e, e'), e < e', no shared vertex, that may lie within `margin`; sorted."""
    Ne = edges.shape[0]
    if Ne * (Ne - 1) // 2 <= BRUTE_LIMIT:
        e, e2 = _ee_all(Ne)
    else:
        mid = 0.5 * (s[edges[:, 0]] + s[edges[:, 1]])
        half = np.max(0.5 * np.linalg.norm(s[edges[:, 1]] - s[edges[:, 0]], axis=1))
        tree = cKDTree(mid)
        pr = tree.query_pairs(r=margin + 2 * half * (1 + 1e-9) + 1e-300, output_type="ndarray")
        pr = np.sort(pr, axis=1)
        e, e2 = pr[:, 0], pr[:, 1]
    share = ((edges[e][:, :, None] == edges[e2][:, None, :]).any(axis=(1, 2)))
    e, e2 = e[~share], e2[~share]
    o = np.lexsort((e2, e))
    return e[o], e2[o]


def pair_points(s, tris, edges, kind, i0, i1):
    """Surface-vertex ids (K,4) and stacked positions Y (K,12) of pairs."""
    if kind == "pt":
        ids = np.concatenate([i0[:, None], tris[i1]], axis=1)
    else:
        ids = np.concatenate([edges[i0], edges[i1]], axis=1)
    return ids, s[ids].reshape(-1, 12)


def pair_distance2(s, tris, edges, kind, i0, i1):
    ids, Y = pair_points(s, tris, edges, kind, i0, i1)
    P = [Y[:, 3 * c:3 * c + 3] for c in range(4)]
    if kind == "pt":
        return D.pt_distance2(*P)
    return D.ee_distance2(*P)


def active_set(s, tris, edges, dh):
    """C = {pairs with d^2 < d_hat^2} as sorted lists + per-pair (type, d^2)."""
    dh2 = dh * dh
    out = {}
    for kind in ("pt", "ee"):
        if kind == "pt":
            i0, i1 = pt_candidates(s, tris, dh * 1.01)
        else:
            i0, i1 = ee_candidates(s, edges, dh * 1.01)
        ty, d2 = pair_distance2(s, tris, edges, kind, i0, i1)
        m = d2 < dh2
        out[kind] = (i0[m], i1[m], ty[m], d2[m])
    return out


def contact_vertex_set(W, mesh_free_pos, C, tris, edges):
    """S: sorted unique free sim vertices in the W-support of C's surface verts."""
    js = []
    if C["pt"][0].size:
        js.append(np.concatenate([C["pt"][0][:, None], tris[C["pt"][1]]], axis=1).ravel())
    if C["ee"][0].size:
        js.append(np.concatenate([edges[C["ee"][0]], edges[C["ee"][1]]], axis=1).ravel())
    if not js:
        return np.zeros(0, dtype=np.int64)
    js = np.unique(np.concatenate(js))
    cols = np.unique(W[js].indices)
    return cols[mesh_free_pos[cols] >= 0]


def barrier_derivatives(mesh, s, C, dh, kappa):
    """Pulled-back barrier gradient (n,3), Hessian (3n x 3n sparse), energy and pair terms."""
    n, Ns = mesh.n, s.shape[0]
    gs = np.zeros((Ns, 3))
    rows, cols, vals = [], [], []
    energy = 0.0
    pairs = {}
    for kind in ("pt", "ee"):
        i0, i1, ty, d2 = C[kind]
        if i0.size == 0:
            pairs[kind] = None
            continue
        ids, Y = pair_points(s, mesh.tris, mesh.edges, kind, i0, i1)
        d, bv, h, Hp = Bm.pair_terms(Y, ty, d2, dh, kappa)
        energy += kappa * float(bv.sum())
        np.add.at(gs, ids.ravel(), h.reshape(-1, 3))
        dof = (3 * ids[:, :, None] + np.arange(3)[None, None, :]).reshape(-1, 12)
        rows.append(np.repeat(dof, 12, axis=1).ravel())
        cols.append(np.tile(dof, (1, 12)).ravel())
        vals.append(Hp.reshape(-1))
        pairs[kind] = dict(ids=ids, d=d, b=bv, h=h, Hp=Hp, types=ty)
    Wk = sp.kron(mesh.W, sp.identity(3), format="csr")              # (3Ns, 3n)
    gB = (mesh.W.T @ gs)                                             # (n, 3)
    if rows:
        Hs = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                           shape=(3 * Ns, 3 * Ns)).tocsr()
        HB = (Wk.T @ Hs @ Wk).tocsr()
    else:
        HB = sp.csr_matrix((3 * n, 3 * n))
    return gB, HB, energy, pairs
