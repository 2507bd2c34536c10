"""O3 canonical primitive distances (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

PAPER.md:88 (section 2.2): "for each primitive pair (vertex-triangle or edge-edge), their
unsigned distance d_k is used to compute a barrier ... activated only when the distance is
smaller than a distance threshold d_0".  The paper gives no distance algorithm; this module
is SURVEY.md 8(c) "Canonical distance routine" written out:
  type: Ericson, Real-Time Collision Detection 5.1.5 (point-triangle regions, book order) and
        5.1.9 (segment-segment, with den = |d1 x d2|^2 from the cross product, s = 0 when
        den <= 1e-20 a e);
  d^2:  the type's closed form (PP, point-line, point-plane, line-line), never the
        closest-point difference;
  operation order: component-wise differences, dots summed x then y then z left to right,
        standard cross-product formula, division last, no FMA (numpy ufuncs round every
        operation separately, which is exactly "no contraction").
All functions are vectorised over a leading pair axis: inputs (K, 3) float64.
"""
from __future__ import annotations

import numpy as np

# type labels (oracle-local enumeration)
PT_A, PT_B, PT_C, PT_AB, PT_AC, PT_BC, PT_FACE = 0, 1, 2, 3, 4, 5, 6
EE_EE, EE_PE_A, EE_PE_B, EE_PE_C, EE_PE_D, EE_PP_AC, EE_PP_AD, EE_PP_BC, EE_PP_BD = \
    7, 8, 9, 10, 11, 12, 13, 14, 15


def _sub(u, v):
    return u - v


def _dot(u, v):
    return (u[..., 0] * v[..., 0] + u[..., 1] * v[..., 1]) + u[..., 2] * v[..., 2]


def _cross(u, v):
    return np.stack([u[..., 1] * v[..., 2] - u[..., 2] * v[..., 1],
                     u[..., 2] * v[..., 0] - u[..., 0] * v[..., 2],
                     u[..., 0] * v[..., 1] - u[..., 1] * v[..., 0]], axis=-1)


# ---- closed forms ---------------------------------------------------
def d2_point_point(p, q):
    r = _sub(p, q)
    return _dot(r, r)


def d2_point_edge(p, a, b):
    """|(a-p) x (b-p)|^2 / |b-a|^2 : point to the line through the edge."""
    c = _cross(_sub(a, p), _sub(b, p))
    e = _sub(b, a)
    return _dot(c, c) / _dot(e, e)


def d2_point_plane(p, a, b, c):
    """((p-a).n)^2 / |n|^2, n = (b-a) x (c-a)."""
    n = _cross(_sub(b, a), _sub(c, a))
    t = _dot(_sub(p, a), n)
    return (t * t) / _dot(n, n)


def d2_line_line(a, b, c, d):
    """((c-a).n)^2 / |n|^2, n = (b-a) x (d-c)."""
    n = _cross(_sub(b, a), _sub(d, c))
    t = _dot(_sub(c, a), n)
    return (t * t) / _dot(n, n)


# ---- type selection ----------------------------------------------------------------------
def pt_type(p, a, b, c):
    """Ericson RTCD 5.1.5 ClosestPtPointTriangle region tests, in the book's order."""
    ab = _sub(b, a)
    ac = _sub(c, a)
    ap = _sub(p, a)
    d1 = _dot(ab, ap)
    d2 = _dot(ac, ap)
    bp = _sub(p, b)
    d3 = _dot(ab, bp)
    d4 = _dot(ac, bp)
    vc = d1 * d4 - d3 * d2
    cp = _sub(p, c)
    d5 = _dot(ab, cp)
    d6 = _dot(ac, cp)
    vb = d5 * d2 - d1 * d6
    va = d3 * d6 - d5 * d4
    conds = [(d1 <= 0) & (d2 <= 0),
             (d3 >= 0) & (d4 <= d3),
             (vc <= 0) & (d1 >= 0) & (d3 <= 0),
             (d6 >= 0) & (d5 <= d6),
             (vb <= 0) & (d2 >= 0) & (d6 <= 0),
             (va <= 0) & ((d4 - d3) >= 0) & ((d5 - d6) >= 0)]
    return np.select(conds, [PT_A, PT_B, PT_AB, PT_C, PT_AC, PT_BC], default=PT_FACE)


def ee_type(a, b, c, d):
    """Ericson RTCD 5.1.9 ClosestPtSegmentSegment for (a,b) vs (c,d) -> type label."""
    d1 = _sub(b, a)
    d2 = _sub(d, c)
    r = _sub(a, c)
    A = _dot(d1, d1)
    E = _dot(d2, d2)
    Fv = _dot(d2, r)
    C = _dot(d1, r)
    Bv = _dot(d1, d2)
    cr = _cross(d1, d2)
    den = _dot(cr, cr)
    nonpar = den > 1e-20 * A * E
    with np.errstate(divide="ignore", invalid="ignore"):
        s = np.where(nonpar, np.clip((Bv * Fv - C * E) / den, 0.0, 1.0), 0.0)
        t = (Bv * s + Fv) / E
        lo = t < 0.0
        hi = t > 1.0
        s = np.where(lo, np.clip(-C / A, 0.0, 1.0), np.where(hi, np.clip((Bv - C) / A, 0.0, 1.0), s))
        t = np.where(lo, 0.0, np.where(hi, 1.0, t))
    s_in = (s > 0.0) & (s < 1.0)
    t_in = (t > 0.0) & (t < 1.0)
    s1 = s >= 1.0          # s in {0,1} when not inside
    t1 = t >= 1.0
    pe_e1 = np.where(s1, EE_PE_B, EE_PE_A)                 # endpoint of edge 1 vs edge 2
    pe_e2 = np.where(t1, EE_PE_D, EE_PE_C)                 # endpoint of edge 2 vs edge 1
    pp = np.where(s1, np.where(t1, EE_PP_BD, EE_PP_BC), np.where(t1, EE_PP_AD, EE_PP_AC))
    return np.select([s_in & t_in, t_in & ~s_in, s_in & ~t_in], [EE_EE, pe_e1, pe_e2],
                     default=pp)


# ---- type + d^2 --------------------------------------------------------------------------
def pt_distance2(p, a, b, c):
    """(type, d^2) for point p vs triangle (a, b, c)."""
    ty = pt_type(p, a, b, c)
    d2 = np.empty(ty.shape)
    for lab, fn in ((PT_A, lambda m: d2_point_point(p[m], a[m])),
                    (PT_B, lambda m: d2_point_point(p[m], b[m])),
                    (PT_C, lambda m: d2_point_point(p[m], c[m])),
                    (PT_AB, lambda m: d2_point_edge(p[m], a[m], b[m])),
                    (PT_AC, lambda m: d2_point_edge(p[m], a[m], c[m])),
                    (PT_BC, lambda m: d2_point_edge(p[m], b[m], c[m])),
                    (PT_FACE, lambda m: d2_point_plane(p[m], a[m], b[m], c[m]))):
        m = ty == lab
        if m.any():
            d2[m] = fn(m)
    return ty, d2


def ee_distance2(a, b, c, d):
    """(type, d^2) for edge (a, b) vs edge (c, d)."""
    ty = ee_type(a, b, c, d)
    d2 = np.empty(ty.shape)
    for lab, fn in ((EE_EE, lambda m: d2_line_line(a[m], b[m], c[m], d[m])),
                    (EE_PE_A, lambda m: d2_point_edge(a[m], c[m], d[m])),
                    (EE_PE_B, lambda m: d2_point_edge(b[m], c[m], d[m])),
                    (EE_PE_C, lambda m: d2_point_edge(c[m], a[m], b[m])),
                    (EE_PE_D, lambda m: d2_point_edge(d[m], a[m], b[m])),
                    (EE_PP_AC, lambda m: d2_point_point(a[m], c[m])),
                    (EE_PP_AD, lambda m: d2_point_point(a[m], d[m])),
                    (EE_PP_BC, lambda m: d2_point_point(b[m], c[m])),
                    (EE_PP_BD, lambda m: d2_point_point(b[m], d[m]))):
        m = ty == lab
        if m.any():
            d2[m] = fn(m)
    return ty, d2
