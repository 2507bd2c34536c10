"""Pins for oracle O3 (distances, active set), O4 (barrier), O5 (contact vertex set).

Independent checks: textbook special cases (tests/golden/pins.json), an exact distance
computed by a different algorithm (face projection / interior critical point + clamped
endpoint-segment minima), closed forms of b, central finite differences, eigen invariants,
brute-force all-pairs enumeration, and a hand-computed S.
"""
import json
import os
import types

import numpy as np
import pytest

import scenes
from oracle import barrier as Bm
from oracle import build_mesh
from oracle import contact as Ct
from oracle import distance as D

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))


def _a(v):
    return np.asarray(v, float)[None]


# ------------------------------------------------------------------ independent distances --
def _pt_seg(p, a, b):
    ab = b - a
    t = np.clip(np.sum((p - a) * ab, -1) / np.sum(ab * ab, -1), 0, 1)
    q = a + t[..., None] * ab
    return np.sum((p - q) ** 2, -1)


def exact_pt(p, a, b, c):
    """min over the face projection (if inside) and the three edges."""
    n = np.cross(b - a, c - a)
    M = np.stack([b - a, c - a, n], -1)
    uvw = np.linalg.solve(M, (p - a)[..., None])[..., 0]
    u, v = uvw[..., 0], uvw[..., 1]
    inside = (u >= 0) & (v >= 0) & (u + v <= 1)
    face = (uvw[..., 2] ** 2) * np.sum(n * n, -1)
    e = np.minimum(np.minimum(_pt_seg(p, a, b), _pt_seg(p, b, c)), _pt_seg(p, a, c))
    return np.where(inside, np.minimum(face, e), e)


def exact_ee(a, b, c, d):
    """min over the interior critical point (if inside) and 4 endpoint-segment distances."""
    u, v, w = b - a, d - c, a - c
    A, B, C = np.sum(u * u, -1), np.sum(u * v, -1), np.sum(v * v, -1)
    Dd, E = np.sum(u * w, -1), np.sum(v * w, -1)
    den = A * C - B * B
    with np.errstate(all="ignore"):
        s = (B * E - C * Dd) / den
        t = (A * E - B * Dd) / den
    ok = (den > 1e-14 * A * C) & (s > 0) & (s < 1) & (t > 0) & (t < 1)
    P = a + np.nan_to_num(s)[..., None] * u
    Q = c + np.nan_to_num(t)[..., None] * v
    inner = np.sum((P - Q) ** 2, -1)
    e = np.minimum(np.minimum(_pt_seg(a, c, d), _pt_seg(b, c, d)),
                   np.minimum(_pt_seg(c, a, b), _pt_seg(d, a, b)))
    return np.where(ok, np.minimum(inner, e), e)


def test_distance_textbook_cases():
    g = GOLD["distance_cases"]
    for key, lab in (("point_above_centroid", D.PT_FACE), ("point_beyond_vertex", D.PT_A),
                     ("point_beyond_edge", D.PT_AB)):
        c = g[key]
        tri = np.array(c["tri"], float)
        ty, d2 = D.pt_distance2(_a(c["p"]), _a(tri[0]), _a(tri[1]), _a(tri[2]))
        assert ty[0] == lab
        assert abs(np.sqrt(d2[0]) - c["d"]) < 1e-14
    for key, lab in (("perpendicular_skew", D.EE_EE), ("parallel_offset", None)):
        c = g[key]
        e1, e2 = np.array(c["e1"], float), np.array(c["e2"], float)
        ty, d2 = D.ee_distance2(_a(e1[0]), _a(e1[1]), _a(e2[0]), _a(e2[1]))
        if lab is not None:
            assert ty[0] == lab
        assert abs(np.sqrt(d2[0]) - c["d"]) < 1e-14


@pytest.mark.parametrize("scale", [1e-3, 1.0, 1e3])
def test_distance_vs_exact(scale):
    rng = np.random.default_rng(11)
    K = 20000
    P = [scale * rng.standard_normal((K, 3)) for _ in range(4)]
    ty, d2 = D.pt_distance2(*P)
    ref = exact_pt(*P)
    assert np.all(np.abs(d2 - ref) <= 1e-9 * ref + 1e-30 * scale ** 2)
    assert set(np.unique(ty)) == set(range(7))             # every PT type exercised
    ty, d2 = D.ee_distance2(*P)
    ref = exact_ee(*P)
    assert np.all(np.abs(d2 - ref) <= 1e-9 * ref + 1e-30 * scale ** 2)
    assert set(np.unique(ty)) == set(range(7, 16))         # every EE type exercised


def test_ee_parallel_uses_cross_product_den():
    # exactly parallel coplanar edges sqrt(2) h apart on a grid plane
    h = 0.01
    a, b = _a([0, 0, 0]), _a([h, h, 0])
    c, d = _a([h, 0, 0]), _a([2 * h, h, 0])
    _, d2 = D.ee_distance2(a, b, c, d)
    assert abs(np.sqrt(d2[0]) - h / np.sqrt(2)) < 1e-15


# ------------------------------------------------------------------ barrier ---------------
def test_barrier_closed_forms():
    g = GOLD["barrier_half_dhat"]
    assert abs(Bm.b(np.array([g["d"]]), g["d_hat"])[0] - g["value"]) < 1e-16
    dh = 0.3
    for f in (Bm.b, Bm.db, Bm.d2b):
        assert f(np.array([dh, 1.5 * dh]), dh).tolist() == [0.0, 0.0]
    d = np.linspace(1e-4, dh * (1 - 1e-6), 100001)
    assert (Bm.db(d, dh) < 0).all() and (Bm.d2b(d, dh) > 0).all()
    h = 1e-7
    d = np.linspace(0.01, 0.29, 57)
    fd1 = (Bm.b(d + h, dh) - Bm.b(d - h, dh)) / (2 * h)
    fd2 = (Bm.db(d + h, dh) - Bm.db(d - h, dh)) / (2 * h)
    assert np.abs(fd1 - Bm.db(d, dh)).max() < 1e-7 * np.abs(Bm.db(d, dh)).max()
    assert np.abs(fd2 - Bm.d2b(d, dh)).max() < 1e-6 * np.abs(Bm.d2b(d, dh)).max()
    # C^2 at d_hat: derivatives -> 0 from below
    assert abs(Bm.db(np.array([dh * (1 - 1e-6)]), dh)[0]) < 1e-9


def _energy(kind, Y, dh, kappa):
    P = [Y[:, 3 * c:3 * c + 3] for c in range(4)]
    _, d2 = (D.pt_distance2 if kind == "pt" else D.ee_distance2)(*P)
    return kappa * Bm.b(np.sqrt(d2), dh)


@pytest.mark.parametrize("kind", ["pt", "ee"])
def test_pair_gradient_hessian_fd(kind):
    rng = np.random.default_rng(21 if kind == "pt" else 22)
    dh, kappa = 1.0, 3.0
    done = 0
    while done < 40:
        Y = rng.uniform(-1, 1, (1, 12))
        P = [Y[:, 3 * c:3 * c + 3] for c in range(4)]
        ty, d2 = (D.pt_distance2 if kind == "pt" else D.ee_distance2)(*P)
        if not (0.05 < d2[0] < 0.8):
            continue
        # stay away from type boundaries: the type must be stable under perturbation
        stable = all((D.pt_distance2 if kind == "pt" else D.ee_distance2)(
            *[(Y + 1e-4 * rng.standard_normal(Y.shape))[:, 3 * c:3 * c + 3] for c in range(4)])[0][0]
            == ty[0] for _ in range(8))
        if not stable:
            continue
        d, bv, h, Hp = Bm.pair_terms(Y, ty, d2, dh, kappa)
        eps = 1e-6
        fd = np.zeros(12)
        for k in range(12):
            Yp, Ym = Y.copy(), Y.copy()
            Yp[0, k] += eps
            Ym[0, k] -= eps
            fd[k] = (_energy(kind, Yp, dh, kappa) - _energy(kind, Ym, dh, kappa))[0] / (2 * eps)
        assert np.abs(fd - h[0]).max() < 1e-6 * np.abs(h[0]).max()
        # unprojected Hessian vs FD of the gradient
        G2, H2 = Bm.d2_derivatives(Y, ty)
        gd = G2 / (2 * d)[:, None]
        Hd = (H2 - 2 * gd[:, :, None] * gd[:, None, :]) / (2 * d)[:, None, None]
        Hk = kappa * (Bm.d2b(d, dh)[:, None, None] * gd[:, :, None] * gd[:, None, :]
                      + Bm.db(d, dh)[:, None, None] * Hd)
        fdH = np.zeros((12, 12))
        for k in range(12):
            Yp, Ym = Y.copy(), Y.copy()
            Yp[0, k] += eps
            Ym[0, k] -= eps
            fdH[:, k] = (Bm.pair_terms(Yp, ty, (D.pt_distance2 if kind == "pt" else D.ee_distance2)(
                *[Yp[:, 3 * c:3 * c + 3] for c in range(4)])[1], dh, kappa)[2][0]
                - Bm.pair_terms(Ym, ty, (D.pt_distance2 if kind == "pt" else D.ee_distance2)(
                    *[Ym[:, 3 * c:3 * c + 3] for c in range(4)])[1], dh, kappa)[2][0]) / (2 * eps)
        assert np.abs(fdH - Hk[0]).max() < 1e-5 * np.abs(Hk[0]).max()
        # PSD projection invariants
        lam = np.linalg.eigvalsh(Hp[0])
        assert lam.min() >= -1e-12 * np.abs(Hk[0]).max()
        assert np.abs(Bm.psd_project(Hp) - Hp).max() < 1e-10 * np.abs(Hp).max()
        done += 1


def test_psd_identity_on_psd_input():
    rng = np.random.default_rng(4)
    M = rng.standard_normal((5, 12, 12))
    H = M @ M.transpose(0, 2, 1)
    assert np.abs(Bm.psd_project(H) - H).max() < 1e-12 * np.abs(H).max()


# ------------------------------------------------------------------ active set -----------
def _contact_state():
    """C1 slabs pushed together: a contact-rich but intersection-free state."""
    from oracle import OracleSolver
    sc = scenes.slabs_c1()
    o = OracleSolver(sc)
    x = sc.rest.copy()
    for _ in range(5):
        x = o.iterate(x, sc.actuation(0))["x"]
    return sc, o, x


@pytest.fixture(scope="module")
def contact_state():
    return _contact_state()


def test_active_set_matches_brute_force(contact_state, monkeypatch):
    sc, o, x = contact_state
    m = o.mesh
    s = m.W @ x
    C = Ct.active_set(s, m.tris, m.edges, sc.d_hat)
    monkeypatch.setattr(Ct, "BRUTE_LIMIT", 10 ** 9)
    Cb = Ct.active_set(s, m.tris, m.edges, sc.d_hat)
    for k in ("pt", "ee"):
        assert np.array_equal(C[k][0], Cb[k][0]) and np.array_equal(C[k][1], Cb[k][1])
    # brute-force definition: every non-incident pair with d^2 < d_hat^2, nothing else
    Ns, Nt = s.shape[0], m.tris.shape[0]
    j, f = np.repeat(np.arange(Ns), Nt), np.tile(np.arange(Nt), Ns)
    keep = ~(m.tris[f] == j[:, None]).any(1)
    _, d2 = Ct.pair_distance2(s, m.tris, m.edges, "pt", j[keep], f[keep])
    assert int((d2 < sc.d_hat ** 2).sum()) == C["pt"][0].size > 0
    assert C["ee"][0].size > 0


def test_gradient_pullback_fd(contact_state):
    sc, o, x = contact_state
    m = o.mesh
    s = m.W @ x
    C = Ct.active_set(s, m.tris, m.edges, sc.d_hat)
    gB, HB, EB, _ = Ct.barrier_derivatives(m, s, C, sc.d_hat, sc.kappa)

    def B(xx):
        ss = m.W @ xx
        CC = Ct.active_set(ss, m.tris, m.edges, sc.d_hat)
        return Ct.barrier_derivatives(m, ss, CC, sc.d_hat, sc.kappa)[2]

    S = Ct.contact_vertex_set(m.W, m.free_pos, C, m.tris, m.edges)
    rng = np.random.default_rng(0)
    eps = 1e-9 * sc.h
    for v in rng.choice(S, 6, replace=False):
        for a in range(3):
            xp, xm = x.copy(), x.copy()
            xp[v, a] += eps
            xm[v, a] -= eps
            fd = (B(xp) - B(xm)) / (2 * eps)
            assert abs(fd - gB[v, a]) < 1e-5 * np.abs(gB).max()


def test_contact_vertex_set_hand_computed():
    """One active PT pair between two single tets; W picks surface verts from the tets.

    Lower tet (0,1,2,3) with vertex 0 fixed; upper tet (4,5,6,7) with vertex 7 fixed.  The
    surface is the lower tet's slanted face (1,2,3) plus vertex 4 of the upper tet, placed
    0.1 above that face's centroid along its normal (d_hat = 0.2).  The only pair is
    (point 3 = sim 4, triangle 0); its 4 surface vertices map to sim {1,2,3,4}, none fixed,
    so S = [1, 2, 3, 4].
    """
    P = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1],
                  [0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
    P[4:] += 1.0 / 3.0 + 0.1 / np.sqrt(3.0)
    T = np.array([[0, 1, 2, 3], [4, 5, 6, 7]], dtype=np.int32)
    # surface vertices: sim 1, 2, 3 (lower face) and sim 4 (point); one triangle (0,1,2)
    et = np.array([0, 0, 0, 1], np.int32)
    ew = np.zeros((4, 4))
    ew[0, 1] = ew[1, 2] = ew[2, 3] = ew[3, 0] = 1.0
    sc = types.SimpleNamespace(rest=P, tets=T, fixed=np.array([0, 7]),
                               surf_tris=np.array([[0, 1, 2]]), embed_tet=et, embed_w=ew)
    m = build_mesh(sc)
    s = m.W @ P
    C = Ct.active_set(s, m.tris, m.edges, 0.2)
    assert C["pt"][0].tolist() == [3] and C["pt"][1].tolist() == [0] and C["ee"][0].size == 0
    S = Ct.contact_vertex_set(m.W, m.free_pos, C, m.tris, m.edges)
    assert S.tolist() == [1, 2, 3, 4]
