"""Pins for the four oracle parts the round-1 review found unpinned (VERDICT r1 "What's weak" 1).

Each test is built so that the plausible mistake named beside it fails:
  * psd_project (O4, "PositiveDefinite"): a 12x12 with a KNOWN
    spectrum built from a random orthogonal Q must map to Q max(Lambda, 0) Q^T exactly, and H^+
    must satisfy the Frobenius-nearest-PSD conditions (H - H^+ negative semidefinite,
    H^+ (H - H^+) = 0) and beat sampled PSD matrices.   Mutation: |lambda| instead of max(.,0).
  * the contact Hessian pull-back (O4, "script-B = W^T hess_s B W"): HB must equal
    an independently looped dense sum_k J_k^T H_k^+ J_k with J_k built from the pair's OWN
    surface vertices (PT: (j, f0, f1, f2); EE: (e0, e1, e'0, e'1)) and the rows of W; with the
    projection switched off, HB must equal central finite differences of the pulled-back
    gradient.  Mutation: stencil with the vertex order reversed.
  * the line search (O8): constructed elastic cases whose
    acceptance threshold is known in closed form give exactly 2 and 5 halvings; an uphill
    direction gives alpha = 0, STALL, 31 trials; on a real contact state the returned energy
    difference equals a brute-force surrogate-energy difference summed over ALL non-incident
    pairs.  Mutations: halving by 3, a cap of 2 halvings.
  * the swept candidate set (O7): must equal an all-pairs enumeration of
    d_hat-inflated swept-box overlaps on C1 with random dx.  Mutation: no d_hat inflation.
"""
import numpy as np
import pytest
import scipy.sparse as sp

import scenes
from oracle import OracleSolver
from oracle import barrier as Bm
from oracle import ccd as Cc
from oracle import contact as Ct
from oracle import distance as D
from oracle.solver import STALL


# ------------------------------------------------------------------ PSD projection --------
def _random_orthogonal(rng, n=12):
    Q, R = np.linalg.qr(rng.standard_normal((n, n)))
    return Q * np.sign(np.diag(R))[None, :]


def test_psd_projection_known_spectrum():
    rng = np.random.default_rng(123)
    lam = np.array([3.0, -2.0, 1e-3, -1e-4, 0.5, -0.7, 2.0, -3e-2, 1e-6, 4.0, -5.0, 0.1])
    Hs, Ps = [], []
    for _ in range(6):
        Q = _random_orthogonal(rng)
        Hs.append(Q @ np.diag(lam) @ Q.T)
        Ps.append(Q @ np.diag(np.maximum(lam, 0.0)) @ Q.T)
    H = np.stack(Hs)
    H = 0.5 * (H + H.transpose(0, 2, 1))
    Hp = Bm.psd_project(H)
    assert np.abs(Hp - np.stack(Ps)).max() < 1e-13 * np.abs(lam).max()
    for k in range(H.shape[0]):
        Dk = H[k] - Hp[k]
        # Frobenius-nearest PSD matrix (Higham 1988): H - H^+ is NSD and orthogonal to H^+
        assert np.linalg.eigvalsh(Dk).max() <= 1e-13 * np.abs(lam).max()
        assert np.abs(Hp[k] @ Dk).max() <= 1e-13 * np.abs(lam).max() ** 2
        assert np.linalg.eigvalsh(Hp[k]).min() >= -1e-13 * np.abs(lam).max()
        # and no sampled PSD matrix is closer to H
        best = np.linalg.norm(Dk)
        assert best == pytest.approx(np.sqrt(np.sum(np.minimum(lam, 0.0) ** 2)), rel=1e-12)
        for _ in range(200):
            M = rng.standard_normal((12, 12)) * rng.uniform(0.01, 1.0)
            P = Hp[k] + 0.05 * M @ M.T
            assert np.linalg.norm(H[k] - P) >= best


# ------------------------------------------------------------------ pull-back -------------
@pytest.fixture(scope="module")
def c1_contact():
    sc = scenes.slabs_c1()
    o = OracleSolver(sc)
    x = sc.rest.copy()
    log = []
    for _ in range(8):
        it = o.iterate(x, sc.actuation(0))
        log.append((x, it))
        x = it["x"]
    return sc, o, log


def _pair_surface_ids(m, kind, i0, i1):
    """Surface-vertex ids of pairs written from the definitions (not via oracle helpers)."""
    out = []
    for a, b in zip(i0.tolist(), i1.tolist()):
        if kind == "pt":
            out.append([a, int(m.tris[b, 0]), int(m.tris[b, 1]), int(m.tris[b, 2])])
        else:
            out.append([int(m.edges[a, 0]), int(m.edges[a, 1]), int(m.edges[b, 0]), int(m.edges[b, 1])])
    return np.array(out, dtype=np.int64).reshape(-1, 4)


def _dense_pullback(m, s, C, Hfun):
    """sum_k J_k^T H_k J_k with J_k = [W_{j_0,:}; ...; W_{j_3,:}] (x) I3, looped pair by pair."""
    n = m.n
    Wd = m.W.toarray()
    HB = np.zeros((3 * n, 3 * n))
    for kind in ("pt", "ee"):
        i0, i1, ty, d2 = C[kind]
        if i0.size == 0:
            continue
        ids = _pair_surface_ids(m, kind, i0, i1)
        Hk = Hfun(s[ids].reshape(-1, 12), ty, d2)
        for k in range(ids.shape[0]):
            J = np.zeros((12, 3 * n))
            for c in range(4):
                for a in range(3):
                    J[3 * c + a, a::3] = Wd[ids[k, c]]
            HB += J.T @ Hk[k] @ J
    return HB


def test_hessian_pullback_independent_loop(c1_contact):
    sc, o, log = c1_contact
    m = o.mesh
    x = log[6][0]
    s = m.W @ x
    C = Ct.active_set(s, m.tris, m.edges, sc.d_hat)
    assert C["pt"][0].size > 50 and C["ee"][0].size > 50
    _, HB, _, _ = Ct.barrier_derivatives(m, s, C, sc.d_hat, sc.kappa)
    ref = _dense_pullback(m, s, C, lambda Y, ty, d2: Bm.pair_terms(Y, ty, d2, sc.d_hat, sc.kappa)[3])
    assert np.abs(HB.toarray() - ref).max() <= 1e-12 * np.abs(ref).max()


def test_hessian_pullback_fd_without_projection(c1_contact, monkeypatch):
    """With the per-pair projection switched off, HB is the exact Jacobian of the pulled-back
    barrier gradient W^T grad_s B: central differences, columns on S."""
    sc, o, log = c1_contact
    m = o.mesh
    x = log[6][0]
    monkeypatch.setattr(Bm, "psd_project", lambda H: H)
    s = m.W @ x
    C = Ct.active_set(s, m.tris, m.edges, sc.d_hat)
    gB, HB, _, _ = Ct.barrier_derivatives(m, s, C, sc.d_hat, sc.kappa)
    HB = HB.toarray()
    S = Ct.contact_vertex_set(m.W, m.free_pos, C, m.tris, m.edges)
    rng = np.random.default_rng(5)
    eps = 1e-8 * sc.h
    scale = np.abs(HB).max()
    for v in rng.choice(S, 8, replace=False):
        for a in range(3):
            cols = []
            for sgn in (1.0, -1.0):
                xx = x.copy()
                xx[v, a] += sgn * eps
                ss = m.W @ xx
                # the same pairs as C (the FD must not cross an activation boundary), their
                # types and distances re-evaluated at the perturbed positions
                Cp = {}
                for kind in ("pt", "ee"):
                    i0, i1 = C[kind][0], C[kind][1]
                    ty, d2 = Ct.pair_distance2(ss, m.tris, m.edges, kind, i0, i1)
                    Cp[kind] = (i0, i1, ty, d2)
                g, _, _, _ = Ct.barrier_derivatives(m, ss, Cp, sc.d_hat, sc.kappa)
                cols.append(g.ravel())
            fd = (cols[0] - cols[1]) / (2 * eps)
            assert np.abs(fd - HB[:, 3 * v + a]).max() < 2e-5 * scale


# ------------------------------------------------------------------ line search -----------
def _pd_scene():
    sc = scenes.slabs_c1()
    return scenes.Scene(sc.name + "_pd", sc.rest, sc.tets, sc.fixed, np.zeros((0, 3), np.int32),
                        np.zeros(0, np.int32), np.zeros((0, 4)), sc.d_hat, sc.kappa, sc.h,
                        sc.n_frames, sc.n_iters, sc.actuation)


def _quad_from_tets(sc, dx):
    """sum_i w_i ||G_i dx||_F^2 written from Eq. 1-2: G_i dx = D_s(dx) D_m^-1, w_i = det D_m / 6."""
    X, T = sc.rest, sc.tets
    q = 0.0
    for t in T:
        Dm = np.column_stack([X[t[1]] - X[t[0]], X[t[2]] - X[t[0]], X[t[3]] - X[t[0]]])
        Ds = np.column_stack([dx[t[1]] - dx[t[0]], dx[t[2]] - dx[t[0]], dx[t[3]] - dx[t[0]]])
        F = Ds @ np.linalg.inv(Dm)
        q += np.linalg.det(Dm) / 6.0 * np.sum(F * F)
    return q


@pytest.mark.parametrize("frac,halvings", [(0.3, 2), (0.05, 5)])
def test_line_search_constructed_halvings(frac, halvings):
    """Elastic-only Delta E(alpha) = alpha g + 1/2 alpha^2 q (Z6/Z7) is < 0 iff alpha < -2g/q.
    With -2g/q = frac * alpha_m the first accepted trial is alpha_m / 2^h with h the smallest
    integer such that 2^-h < frac."""
    sc = _pd_scene()
    o = OracleSolver(sc)
    m = o.mesh
    rng = np.random.default_rng(77)
    dx = np.zeros((m.n, 3))
    dx[m.free] = rng.standard_normal((m.n_free, 3)) * 1e-3
    q = _quad_from_tets(sc, dx)
    am = 0.8
    g = -0.5 * frac * am * q                      # -2g/q = frac * am
    g_el = np.zeros((m.n, 3))
    g_el[m.free] = dx[m.free] * (g / np.sum(dx[m.free] ** 2))
    alpha, trials, flags, dE = o.line_search(sc.rest.copy(), None, dx, None, g_el, None, am)
    assert flags == 0 and trials == halvings + 1
    assert alpha == am / 2 ** halvings
    assert dE == pytest.approx(alpha * g + 0.5 * alpha * alpha * q, rel=1e-10)
    assert dE < 0


def test_line_search_uphill_stalls():
    sc = _pd_scene()
    o = OracleSolver(sc)
    m = o.mesh
    rng = np.random.default_rng(78)
    dx = np.zeros((m.n, 3))
    dx[m.free] = rng.standard_normal((m.n_free, 3)) * 1e-3
    g_el = dx.copy()                              # g^T dx > 0: every alpha > 0 increases E
    alpha, trials, flags, dE = o.line_search(sc.rest.copy(), None, dx, None, g_el, None, 1.0)
    assert alpha == 0.0 and flags == STALL and trials == 31 and dE == 0.0


def _all_pairs_barrier(m, s, dh, kappa):
    """kappa sum over ALL non-incident PT and EE pairs of b(d) (brute force)."""
    Ns, Nt, Ne = s.shape[0], m.tris.shape[0], m.edges.shape[0]
    j, f = np.repeat(np.arange(Ns), Nt), np.tile(np.arange(Nt), Ns)
    keep = ~(m.tris[f] == j[:, None]).any(1)
    _, d2 = D.pt_distance2(s[j[keep]], s[m.tris[f[keep], 0]], s[m.tris[f[keep], 1]], s[m.tris[f[keep], 2]])
    e, e2 = np.triu_indices(Ne, k=1)
    keep = ~(m.edges[e][:, :, None] == m.edges[e2][:, None, :]).any(axis=(1, 2))
    e, e2 = e[keep], e2[keep]
    _, d2e = D.ee_distance2(s[m.edges[e, 0]], s[m.edges[e, 1]], s[m.edges[e2, 0]], s[m.edges[e2, 1]])
    return kappa * (Bm.b(np.sqrt(d2), dh).sum() + Bm.b(np.sqrt(d2e), dh).sum())


def _elastic_surrogate(sc, x, p):
    """1/2 sum_i w_i ||F_i(x) - P_i||_F^2 with P fixed (Z6/Z7), written from the tets."""
    X, T = sc.rest, sc.tets
    E = 0.0
    for i, t in enumerate(T):
        Dm = np.column_stack([X[t[1]] - X[t[0]], X[t[2]] - X[t[0]], X[t[3]] - X[t[0]]])
        Ds = np.column_stack([x[t[1]] - x[t[0]], x[t[2]] - x[t[0]], x[t[3]] - x[t[0]]])
        R = Ds @ np.linalg.inv(Dm) - p[i].reshape(3, 3)
        E += 0.5 * np.linalg.det(Dm) / 6.0 * np.sum(R * R)
    return E


def test_line_search_energy_matches_all_pairs_brute_force(c1_contact):
    sc, o, log = c1_contact
    m = o.mesh
    checked = 0
    for x0, it in log[2:6]:
        x1 = it["x"]
        dE_bf = (_elastic_surrogate(sc, x1, it["p"]) - _elastic_surrogate(sc, x0, it["p"])
                 + _all_pairs_barrier(m, m.W @ x1, sc.d_hat, sc.kappa)
                 - _all_pairs_barrier(m, m.W @ x0, sc.d_hat, sc.kappa))
        assert it["dE"] < 0
        assert abs(it["dE"] - dE_bf) <= 1e-7 * abs(it["dE"])
        checked += 1
    assert checked == 4


# ------------------------------------------------------------------ swept pairs -----------
def _swept_all_pairs(s, ds, tris, edges, dh):
    s1 = s + ds
    lo, hi = np.minimum(s, s1), np.maximum(s, s1)

    def box(ids):
        return lo[ids].min(axis=1) - dh, hi[ids].max(axis=1) + dh

    Ns, Nt, Ne = s.shape[0], tris.shape[0], edges.shape[0]
    j, f = np.repeat(np.arange(Ns), Nt), np.tile(np.arange(Nt), Ns)
    keep = ~(tris[f] == j[:, None]).any(1)
    j, f = j[keep], f[keep]
    la, ha = box(j[:, None])
    lb, hb = box(tris[f])
    ov = ((la <= hb) & (lb <= ha)).all(1)
    pt = (j[ov], f[ov])
    e, e2 = np.triu_indices(Ne, k=1)
    keep = ~(edges[e][:, :, None] == edges[e2][:, None, :]).any(axis=(1, 2))
    e, e2 = e[keep], e2[keep]
    la, ha = box(edges[e])
    lb, hb = box(edges[e2])
    ov = ((la <= hb) & (lb <= ha)).all(1)
    return {"pt": pt, "ee": (e[ov], e2[ov])}


def test_swept_pairs_equal_all_pairs_enumeration(c1_contact):
    sc, o, log = c1_contact
    m = o.mesh
    rng = np.random.default_rng(31)
    for k, scale in ((3, 0.05), (5, 0.3), (7, 1.0)):
        s = m.W @ log[k][0]
        ds = rng.standard_normal(s.shape) * scale * sc.h
        sw = Cc.swept_pairs(s, ds, m.tris, m.edges, sc.d_hat)
        bf = _swept_all_pairs(s, ds, m.tris, m.edges, sc.d_hat)
        for kind in ("pt", "ee"):
            a = np.stack(sw[kind], 1)
            b = np.stack(bf[kind], 1)
            b = b[np.lexsort((b[:, 1], b[:, 0]))]
            assert a.shape[0] > 0 and np.array_equal(a, b), kind


# ------------------------------------------------------------------ low-rank Sigma_s update --
@pytest.mark.parametrize("n_rm, n_add", [(0, 5), (7, 0), (4, 9), (64, 64)])
def test_sigma_update_identities(n_rm, n_add):
    """The two identities the CUDA path's low-rank update of Sigma_s = K_s^-1 rests on (DESIGN.md
    5.3; exact in exact arithmetic), checked against direct inverses of a random SPD K on the
    union of old and new vertex sets: removal Sigma' = Sigma_kk - Sigma_kR Sigma_RR^-1 Sigma_Rk;
    addition with b = K[keep, A], X = Sigma' b, Sc = K[A, A] - b^T X:
    Sigma_new = [[Sigma' + X Sc^-1 X^T, -X Sc^-1], [-Sc^-1 X^T, Sc^-1]]."""
    rng = np.random.default_rng(7 + n_rm + 100 * n_add)
    n_keep = 150
    N = n_keep + n_rm + n_add
    Q = rng.standard_normal((N, N))
    K = Q @ Q.T / N + 0.5 * np.eye(N)
    perm = rng.permutation(N)
    keep, rem, add = perm[:n_keep], perm[n_keep:n_keep + n_rm], perm[n_keep + n_rm:]
    old = np.concatenate([keep, rem])
    Sig_old = np.linalg.inv(K[np.ix_(old, old)])
    k, r = np.arange(n_keep), np.arange(n_keep, n_keep + n_rm)
    Sig_p = Sig_old[np.ix_(k, k)]
    if n_rm:
        Sig_p = Sig_p - Sig_old[np.ix_(k, r)] @ np.linalg.solve(Sig_old[np.ix_(r, r)], Sig_old[np.ix_(r, k)])
    assert np.allclose(Sig_p, np.linalg.inv(K[np.ix_(keep, keep)]), rtol=1e-10, atol=1e-12)
    new = np.concatenate([keep, add])
    if n_add:
        b = K[np.ix_(keep, add)]
        X = Sig_p @ b
        Sc = K[np.ix_(add, add)] - b.T @ X
        Sci = np.linalg.inv(Sc)
        top = np.hstack([Sig_p + X @ Sci @ X.T, -X @ Sci])
        bot = np.hstack([-Sci @ X.T, Sci])
        Sig_new = np.vstack([top, bot])
    else:
        Sig_new = Sig_p
    assert np.allclose(Sig_new, np.linalg.inv(K[np.ix_(new, new)]), rtol=1e-10, atol=1e-12)
