"""Pins for oracle O6 (full solve), O7 (ACCD), O8 (line search) and end-to-end invariants.

Independent checks: the pure-PD global step of Eq. 2 (closed form), the energy decrease
-1/2 g^T H^-1 g, the paper's reduced solves (Eq. 7-8 Schur, Eq. 11 Woodbury, the K-Schur
panel form the CUDA path uses) written out with dense numpy linear algebra, the hand-derived
ACCD head-on case, brute-force intersection tests, quiescence.
"""
import json
import os
import types

import numpy as np
import pytest

import scenes
from oracle import OracleSolver
from oracle import ccd as Cc
from oracle import contact as Ct
from oracle import distance as D

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))


def _no_surface(sc):
    return scenes.Scene(sc.name + "_pd", sc.rest, sc.tets, sc.fixed, np.zeros((0, 3), np.int32),
                        np.zeros(0, np.int32), np.zeros((0, 4)), sc.d_hat, sc.kappa, sc.h,
                        sc.n_frames, sc.n_iters, sc.actuation)


@pytest.fixture(scope="module")
def c1_run():
    sc = scenes.slabs_c1()
    o = OracleSolver(sc)
    log = []
    o.run_frame(sc.rest.copy(), sc.actuation(0), sc.n_iters, log)
    return sc, o, log


# ------------------------------------------------------------------ brute-force crossing --
def edge_triangle_crossings(s, tris, edges):
    """Number of (edge, triangle) pairs, not sharing a vertex, whose segment pierces the
    triangle (Moller-Trumbore, closed test).  Independent of the oracle's distance code."""
    E, T = edges.shape[0], tris.shape[0]
    e = np.repeat(np.arange(E), T)
    t = np.tile(np.arange(T), E)
    share = (edges[e][:, :, None] == tris[t][:, None, :]).any(axis=(1, 2))
    e, t = e[~share], t[~share]
    O = s[edges[e, 0]]
    Dv = s[edges[e, 1]] - O
    v0, v1, v2 = s[tris[t, 0]], s[tris[t, 1]], s[tris[t, 2]]
    e1, e2 = v1 - v0, v2 - v0
    pv = np.cross(Dv, e2)
    det = np.sum(e1 * pv, 1)
    # skip (near-)coplanar configurations: rounding makes det tiny but nonzero there, and a
    # coplanar touch would show up as a zero distance in the distance-based checks anyway
    scale = np.linalg.norm(Dv, axis=1) * np.linalg.norm(np.cross(e1, e2), axis=1)
    ok = np.abs(det) > 1e-10 * scale
    inv = np.where(ok, 1.0 / np.where(ok, det, 1.0), 0.0)
    tv = O - v0
    u = np.sum(tv * pv, 1) * inv
    qv = np.cross(tv, e1)
    v = np.sum(Dv * qv, 1) * inv
    w = np.sum(e2 * qv, 1) * inv
    hit = ok & (u >= 0) & (v >= 0) & (u + v <= 1) & (w >= 0) & (w <= 1)
    return int(hit.sum())


# ------------------------------------------------------------------ O6 / O8 -------------
def test_pure_pd_step_is_eq2_global_step():
    sc = _no_surface(scenes.slabs_c1())
    o = OracleSolver(sc)
    m = o.mesh
    x = sc.rest.copy()
    it = o.iterate(x, sc.actuation(0))
    assert it["alpha_m"] == 1.0 and it["alpha"] == 1.0 and it["ls_trials"] == 1
    # Eq. 2: H x_new = sum w G^T p on free DOFs, i.e. the elastic gradient at x_new with the
    # SAME p vanishes (H x_new - rhs = 0)
    from oracle.local import elastic_gradient
    g_new = elastic_gradient(m, it["x"], it["p"])[m.free]
    assert np.abs(g_new).max() < 1e-10 * np.abs(it["g_el"][m.free]).max()
    # dE(1) = g^T dx + 1/2 dx^T H dx = -1/2 g^T H^-1 g
    gT = it["ghat"]
    Hd = o.H_free.toarray()
    ref = -0.5 * gT @ np.linalg.solve(Hd, gT)
    assert abs(it["dE"] - ref) < 1e-9 * abs(ref)


def test_quiescence_identity_actuation():
    sc = scenes.slabs_c1()
    o = OracleSolver(sc)
    A = np.tile(np.eye(3).reshape(1, 9), (sc.n_tets, 1))
    x = sc.rest.copy()
    for _ in range(3):
        it = o.iterate(x, A)
        assert it["n_pt"] == 0 and it["n_ee"] == 0
        x = it["x"]
    assert np.abs(x - sc.rest).max() < 1e-12 * sc.bbox_diag()


def test_reduced_solves_equal_full_solve(c1_run):
    """Eq. 7-8 (Schur on the W-touched region), Eq. 11 (Woodbury) and the K-Schur panel form
     all reproduce the oracle's full solve on a real contact state."""
    sc, o, log = c1_run
    m = o.mesh
    it = log[5]
    x = log[4]["x"]
    S = it["S"]
    assert S.size > 50
    nf = m.n_free
    Lff = m.Lap[m.free][:, m.free].toarray()
    Hb = o.H_free.toarray()
    ghat = it["ghat"]
    # contact Hessian on free DOFs, rebuilt from the oracle's pair terms
    s = m.W @ x
    C = Ct.active_set(s, m.tris, m.edges, sc.d_hat)
    _, HB, _, _ = Ct.barrier_derivatives(m, s, C, sc.d_hat, sc.kappa)
    HBf = HB[o.free_dof][:, o.free_dof].toarray()
    dx_full = it["dx"][m.free].ravel()
    assert np.abs((Hb + HBf) @ dx_full + ghat).max() < 1e-10 * np.abs(ghat).max()
    fpos = m.free_pos[S]
    Sd = (3 * fpos[:, None] + np.arange(3)).ravel()
    Bc = HBf[np.ix_(Sd, Sd)]
    assert np.abs(HBf).sum() == pytest.approx(np.abs(Bc).sum(), rel=1e-13)   # B lives on S
    # --- K-Schur panel form (what the CUDA path computes)
    Lc = np.linalg.cholesky(Lff)
    E = np.zeros((nf, S.size))
    E[fpos, np.arange(S.size)] = 1.0
    V = np.linalg.solve(Lc, E)                       # panel L^-1 P_S
    G = ghat.reshape(nf, 3)
    w = np.linalg.solve(Lc, G)                       # forward solve, 3 RHS
    yS = -(V.T @ w)                                  # y_S without a backward solve
    Ks = V.T @ V
    Sig = np.linalg.inv(Ks)                          # Schur complement of L onto S
    Sh = np.kron(Sig, np.eye(3)) + Bc
    u = np.linalg.solve(Sh, np.kron(Sig, np.eye(3)) @ yS.ravel())
    t = (Bc @ u).reshape(-1, 3)
    dx_k = -np.linalg.solve(Lc.T, w + V @ t).ravel()
    rel = np.abs(dx_k - dx_full).max() / np.abs(dx_full).max()
    assert rel < 1e-10
    assert np.abs(u - dx_full[Sd]).max() < 1e-10 * np.abs(dx_full).max()
    # --- Eq. 6-8: region x2 = all W-touched free vertices, Schur complement of H11
    reg = np.unique(m.W.indices)
    reg = reg[m.free_pos[reg] >= 0]
    r2 = (3 * m.free_pos[reg][:, None] + np.arange(3)).ravel()
    r1 = np.setdiff1d(np.arange(3 * nf), r2)
    Hh = Hb + HBf
    H11, H12, H22 = Hh[np.ix_(r1, r1)], Hh[np.ix_(r1, r2)], Hh[np.ix_(r2, r2)]
    L1 = np.linalg.cholesky(H11)
    Z = np.linalg.solve(L1, H12)
    Sigh = H22 - Z.T @ Z                             # Eq. 8 (includes B_22)
    y1 = np.linalg.solve(L1, -ghat[r1])              # lower
    z2 = np.linalg.solve(Sigh, -ghat[r2] - Z.T @ y1)  # diagonal (Schur)
    z1 = np.linalg.solve(L1.T, y1 - Z @ z2)          # upper
    dx_s = np.zeros(3 * nf)
    dx_s[r1], dx_s[r2] = z1, z2
    assert np.abs(dx_s - dx_full).max() < 1e-10 * np.abs(dx_full).max()
    # --- Eq. 11 Woodbury on an invertible B (B + 0.1 I; B itself is singular)
    Sig0 = Hb[np.ix_(r2, r2)] - (np.linalg.solve(L1, Hb[np.ix_(r1, r2)])).T @ np.linalg.solve(
        L1, Hb[np.ix_(r1, r2)])
    pos = {v: i for i, v in enumerate(reg)}
    qi = np.array([3 * pos[v] + a for v in S for a in range(3)])
    Q = np.zeros((qi.size, r2.size))
    Q[np.arange(qi.size), qi] = 1.0
    Breg = Bc + 0.1 * np.eye(Bc.shape[0])
    Si = np.linalg.inv(Sig0)
    wood = Si - Si @ Q.T @ np.linalg.inv(np.linalg.inv(Breg) + Q @ Si @ Q.T) @ Q @ Si
    direct = np.linalg.inv(Sig0 + Q.T @ Breg @ Q)
    assert np.abs(wood - direct).max() < 1e-9 * np.abs(direct).max()
    assert np.linalg.matrix_rank(Bc) < Bc.shape[0]                # singular on real data


# ------------------------------------------------------------------ O7 ------------------
def test_accd_head_on_hand_derived():
    g = GOLD["accd_head_on"]
    tri = np.array(g["triangle"], float)
    Y0 = np.concatenate([g["point"], tri.ravel()])[None]
    dY = np.concatenate([g["point_step"], np.zeros(9)])[None]
    toi, its = Cc.accd("pt", Y0, dY)
    assert toi[0] == pytest.approx(g["toi"], abs=1e-15) and its[0] == g["iterations"]
    assert toi[0] < 0.5                                       # analytic contact at 0.5


def test_accd_zero_motion_and_alpha_max():
    sc = scenes.slabs_c1()
    o = OracleSolver(sc)
    m = o.mesh
    s = m.W @ sc.rest
    am, _ = Cc.alpha_max(s, np.zeros_like(s), m.tris, m.edges, sc.d_hat)
    assert am == 1.0


def test_accd_random_perturbations_stay_separated(c1_run):
    sc, o, log = c1_run
    m = o.mesh
    x = log[8]["x"]
    s = m.W @ x
    rng = np.random.default_rng(9)
    free_s = np.asarray((m.W[:, m.free].sum(axis=1) > 0)).ravel()
    for trial in range(40):
        ds = np.zeros_like(s)
        ds[free_s] = rng.standard_normal((int(free_s.sum()), 3)) * sc.h * 0.3
        am, sw = Cc.alpha_max(s, ds, m.tris, m.edges, sc.d_hat)
        assert 0 < am <= 1
        s1 = s + am * ds
        C = Ct.active_set(s1, m.tris, m.edges, sc.d_hat)
        for k in ("pt", "ee"):
            assert (C[k][3] > 0).all()                    # every distance stays > 0
        if trial < 5:
            assert edge_triangle_crossings(s1, m.tris, m.edges) == 0


# ------------------------------------------------------------------ end to end ----------
def test_c1_trajectory_invariants(c1_run):
    sc, o, log = c1_run
    m = o.mesh
    n_c = [len(it["S"]) for it in log]
    n_C = [it["n_pt"] + it["n_ee"] for it in log]
    assert n_C[0] == 0 and max(n_C) > 300 and 100 < n_c[-1] < 250
    for it in log:
        assert it["flags"] == 0 and it["dE"] < 0 and 0 < it["alpha"] <= it["alpha_m"] <= 1
        s = m.W @ it["x"]
        assert edge_triangle_crossings(s, m.tris, m.edges) == 0
    fixed = m.fixed
    assert np.abs(log[-1]["x"][fixed] - sc.rest[fixed]).max() == 0.0


def test_pure_pd_interpenetrates():
    """Without the contact surface the C1 slabs pass through each other, so the contact
    path is what keeps them apart."""
    sc = scenes.slabs_c1()
    o = OracleSolver(_no_surface(sc))
    x = sc.rest.copy()
    for _ in range(30):
        x = o.iterate(x, sc.actuation(0))["x"]
    m_full = OracleSolver(sc).mesh
    s = m_full.W @ x
    assert edge_triangle_crossings(s, m_full.tris, m_full.edges) > 0
