"""O7 continuous collision detection (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

PAPER.md:99, :115 (section 2.2, Alg. 1): "CCD is used to find the largest possible step size
that does not cause penetration"; alpha_m <- CCD(x, dx).  The paper names no algorithm;
SURVEY.md Z9 / 8(c) O7 reading: additive conservative advancement (ACCD) per swept candidate,
s_gap = 0.1, advance factor 0.9, t_max = 1, iteration cap accd_max_iters:
  1. p_i <- Delta_i - mean(Delta) over the pair's 4 points
  2. l_p = max|p| over side 1 + max|p| over side 2 (PT: point | triangle; EE: edge | edge);
     l_p = 0 => TOI = 1
  3. d_init = d(s); g = s_gap d_init; t = 0; t_l = (1 - s_gap) d_init / l_p
  4. loop: d = d(s + (t + t_l) Delta); exit if (t > 0 and d < g) or t + t_l > t_max;
     else t += t_l, t_l = 0.9 d / l_p;  at most accd_max_iters iterations
  5. TOI = t on a gap exit or the cap, else t_max.
alpha_m = min(1, min TOI).  Swept candidates: every non-incident pair whose
AABBs over [s, s + W dx], each inflated by d_hat, overlap.
"""
from __future__ import annotations

import numpy as np
from scipy.spatial import cKDTree

from . import contact as Ct
from . import distance as D


def _box_pairs(lo_a, hi_a, lo_b, hi_b, same):
    """All (a, b) whose boxes overlap (closed test).  A k-d tree on box centres prunes pairs
    whose circumscribed spheres are disjoint, which is exact: overlapping boxes have
    intersecting circumscribed spheres."""
    ca, cb = 0.5 * (lo_a + hi_a), 0.5 * (lo_b + hi_b)
    ra = 0.5 * np.linalg.norm(hi_a - lo_a, axis=1)
    rb = 0.5 * np.linalg.norm(hi_b - lo_b, axis=1)
    if lo_a.shape[0] == 0 or lo_b.shape[0] == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    tree = cKDTree(cb)
    lists = tree.query_ball_point(ca, r=(ra + rb.max()) * (1 + 1e-9) + 1e-300)
    a = np.repeat(np.arange(ca.shape[0]), [len(l) for l in lists])
    b = np.concatenate([np.asarray(l, dtype=np.int64) for l in lists])
    if same:
        keep = a < b
        a, b = a[keep], b[keep]
    ov = ((lo_a[a] <= hi_b[b]) & (lo_b[b] <= hi_a[a])).all(axis=1)
    return a[ov], b[ov]


def swept_pairs(s, ds, tris, edges, dh):
    """Non-incident PT / EE pairs whose d_hat-inflated swept boxes overlap (sorted lists)."""
    s1 = s + ds
    lo = np.minimum(s, s1)
    hi = np.maximum(s, s1)
    out = {}
    # point boxes, triangle boxes, edge boxes, each inflated by d_hat
    lp_, hp_ = lo - dh, hi + dh
    lt = lo[tris].min(axis=1) - dh
    ht = hi[tris].max(axis=1) + dh
    le = lo[edges].min(axis=1) - dh
    he = hi[edges].max(axis=1) + dh
    j, f = _box_pairs(lp_, hp_, lt, ht, same=False)
    inc = (tris[f] == j[:, None]).any(axis=1)
    j, f = j[~inc], f[~inc]
    o = np.lexsort((f, j))
    out["pt"] = (j[o], f[o])
    e, e2 = _box_pairs(le, he, le, he, same=True)
    share = (edges[e][:, :, None] == edges[e2][:, None, :]).any(axis=(1, 2))
    e, e2 = e[~share], e2[~share]
    o = np.lexsort((e2, e))
    out["ee"] = (e[o], e2[o])
    return out


def _dist(kind, P):
    if kind == "pt":
        _, d2 = D.pt_distance2(*P)
    else:
        _, d2 = D.ee_distance2(*P)
    return np.sqrt(d2)


def accd(kind, Y0, dY, s_gap=0.1, t_max=1.0, max_iters=10_000):
    """Vectorised ACCD over pairs: Y0, dY (K, 12) -> TOI (K,), iterations (K,)."""
    K = Y0.shape[0]
    P0 = [Y0[:, 3 * c:3 * c + 3] for c in range(4)]
    Dl = [dY[:, 3 * c:3 * c + 3] for c in range(4)]
    mean = (Dl[0] + Dl[1] + Dl[2] + Dl[3]) / 4.0
    nrm = [np.linalg.norm(Dl[c] - mean, axis=1) for c in range(4)]
    if kind == "pt":
        lp = nrm[0] + np.maximum(np.maximum(nrm[1], nrm[2]), nrm[3])
    else:
        lp = np.maximum(nrm[0], nrm[1]) + np.maximum(nrm[2], nrm[3])
    toi = np.full(K, t_max)
    iters = np.zeros(K, dtype=np.int64)
    act = lp > 0.0
    d_init = _dist(kind, P0)
    g = s_gap * d_init
    t = np.zeros(K)
    with np.errstate(divide="ignore", invalid="ignore"):
        tl = (1.0 - s_gap) * d_init / lp
    idx = np.nonzero(act)[0]
    it = 0
    while idx.size and it < max_iters:
        tt = t[idx] + tl[idx]
        P = [P0[c][idx] + tt[:, None] * Dl[c][idx] for c in range(4)]
        d = _dist(kind, P)
        iters[idx] += 1
        gap_exit = (t[idx] > 0) & (d < g[idx])
        over = tt > t_max
        done = gap_exit | over
        toi[idx[gap_exit]] = t[idx[gap_exit]]
        toi[idx[over & ~gap_exit]] = t_max
        keep = ~done
        k = idx[keep]
        t[k] = tt[keep]
        tl[k] = 0.9 * d[keep] / lp[k]
        idx = k
        it += 1
    toi[idx] = t[idx]                       # iteration cap
    return toi, iters


def alpha_max(s, ds, tris, edges, dh, s_gap=0.1, max_iters=10_000):
    """alpha_m = min(1, min over swept candidates of ACCD TOI) + the swept pair lists."""
    sw = swept_pairs(s, ds, tris, edges, dh)
    am = 1.0
    for kind in ("pt", "ee"):
        i0, i1 = sw[kind]
        if i0.size == 0:
            continue
        ids, Y0 = Ct.pair_points(s, tris, edges, kind, i0, i1)
        dY = ds[ids].reshape(-1, 12)
        toi, _ = accd(kind, Y0, dY, s_gap=s_gap, max_iters=max_iters)
        am = min(am, float(toi.min()))
    return am, sw
