"""Pins for oracle O0 (setup), O1 (local step) and O2 (elastic gradient).

Each test checks the oracle against something other than itself: closed forms, an
independently formulated deformation map, brute-force rotation search, finite differences.
"""
import json
import os
import types

import numpy as np
import pytest

import scenes
from oracle import build_mesh
from oracle.local import elastic_energy, elastic_gradient, local_step, polar_rotation

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))


def _rot(axis, ang):
    axis = np.asarray(axis, float) / np.linalg.norm(axis)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + np.sin(ang) * K + (1 - np.cos(ang)) * K @ K


def _grid_scene(nx, ny, nz, h, fixed_k0=True):
    P, T, cot, ijk = scenes.cube_grid(nx, ny, nz, h)
    fixed = np.nonzero(ijk[:, 2] == 0)[0] if fixed_k0 else np.zeros(0, int)
    return types.SimpleNamespace(rest=P, tets=T, fixed=fixed, surf_tris=np.zeros((0, 3), int),
                                 embed_tet=np.zeros(0, int), embed_w=np.zeros((0, 4)))


def _F_alt(X, tets, x):
    """Deformation gradient with vertex 3 as the origin: F = D_s' D_m'^{-1} (independent form)."""
    Xt, xt = X[tets], x[tets]
    Dm = np.stack([Xt[:, 0] - Xt[:, 3], Xt[:, 1] - Xt[:, 3], Xt[:, 2] - Xt[:, 3]], axis=2)
    Ds = np.stack([xt[:, 0] - xt[:, 3], xt[:, 1] - xt[:, 3], xt[:, 2] - xt[:, 3]], axis=2)
    return np.linalg.solve(Dm.transpose(0, 2, 1), Ds.transpose(0, 2, 1)).transpose(0, 2, 1)


# ---------------------------------------------------------------- O0 -----------------------
def test_rest_deformation_gradient_is_identity():
    sc = scenes.slabs_c1()
    m = build_mesh(sc)
    F = m.deformation_gradients(sc.rest)
    assert np.abs(F - np.eye(3)).max() < 1e-12          # SPEC.md:32 G_i X = vec(I)


def test_volume_closed_form():
    # un-jittered 3x2x2 grid of cubes with h = 0.5 has volume 12 * 0.125 = 1.5 exactly
    m = build_mesh(_grid_scene(3, 2, 2, 0.5))
    assert abs(m.w.sum() - 1.5) < 1e-12 and (m.w > 0).all()


def test_laplacian_invariants():
    sc = scenes.slabs_c1()
    m = build_mesh(sc)
    L = m.Lap
    assert abs(L - L.T).max() < 1e-15
    ones = np.ones(m.n)
    assert np.abs(L @ ones).max() < 1e-12 * abs(L).max()   # translations are in the nullspace
    Lff = L[m.free][:, m.free].toarray()
    assert np.linalg.eigvalsh(Lff).min() > 0               # SPD after Dirichlet elimination


def test_H_matches_independent_dense_assembly():
    sc = scenes.two_tets()
    m = build_mesh(sc)
    n = m.n
    # G_i columns from the independently formulated F (vertex-3 origin), H = sum w G^T G
    H = np.zeros((3 * n, 3 * n))
    for i in range(2):
        G = np.zeros((9, 3 * n))
        for k in range(3 * n):
            e = np.zeros(3 * n)
            e[k] = 1.0
            G[:, k] = _F_alt(sc.rest, sc.tets[i:i + 1], e.reshape(n, 3))[0].reshape(9)
        H += m.w[i] * G.T @ G
    assert np.abs(H - np.kron(m.Lap.toarray(), np.eye(3))).max() < 1e-12 * np.abs(H).max()


def test_setup_errors():
    with pytest.raises(ValueError):
        build_mesh(_grid_scene(2, 1, 1, 1.0, fixed_k0=False))      # no Dirichlet set
    sc = _grid_scene(1, 1, 1, 1.0)
    sc.tets = sc.tets.copy()
    sc.tets[0, [2, 3]] = sc.tets[0, [3, 2]]                        # invert one tet
    with pytest.raises(ValueError):
        build_mesh(sc)


def test_surface_W_reproduces_embedding():
    sc = scenes.face_small()
    m = build_mesh(sc)
    s = m.W @ sc.rest
    # barycentric blend computed independently from host tets and weights
    ref = np.einsum("sc,scd->sd", sc.embed_w, sc.rest[sc.tets[sc.embed_tet]])
    assert np.abs(s - ref).max() < 1e-15
    assert np.abs(np.asarray(m.W.sum(axis=1)).ravel() - 1).max() < 1e-12


# ---------------------------------------------------------------- O1 -----------------------
def test_rigid_motion_identity_actuation():
    sc = scenes.slabs_c1()
    m = build_mesh(sc)
    R0 = _rot([0.3, -0.5, 0.8], 0.7)
    x = sc.rest @ R0.T + np.array([0.1, -0.2, 0.05])
    A = np.tile(np.eye(3).reshape(1, 9), (sc.n_tets, 1))
    p = local_step(m, x, A)
    assert np.abs(p - R0.reshape(1, 9)).max() < 1e-12          # p_i = vec(R0)
    assert elastic_energy(m, x, p) < 1e-24                      # E_i = 0 (north_star pin)


def test_polar_closed_forms():
    g = GOLD["polar_reflection"]
    R = polar_rotation(np.array(g["M"], float)[None])[0]
    assert np.abs(R - np.array(g["R"], float)).max() < 1e-14
    R0 = _rot([1, 2, 3], 1.1)
    R = polar_rotation((R0 @ np.diag([3.0, 2.0, 1.0]))[None])[0]
    assert np.abs(R - R0).max() < 1e-13
    # negative determinant: M = R0 diag(3, 2, -1) -> R0 (flip the smallest axis)
    R = polar_rotation((R0 @ np.diag([3.0, 2.0, -1.0]))[None])[0]
    assert np.abs(R - R0).max() < 1e-13


def test_polar_beats_random_rotations():
    rng = np.random.default_rng(5)
    q = rng.standard_normal((20000, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    Rs = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w),
                   2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w),
                   2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)], 1).reshape(-1, 3, 3)
    for trial in range(6):
        M = rng.standard_normal((3, 3))
        if trial % 2:
            M[:, 0] *= -1.0                                         # det < 0 case
        R = polar_rotation(M[None])[0]
        assert abs(np.linalg.det(R) - 1) < 1e-12 and np.abs(R.T @ R - np.eye(3)).max() < 1e-12
        best = np.min(np.sum((M[None] - Rs) ** 2, axis=(1, 2)))
        assert np.sum((M - R) ** 2) <= best + 1e-12


# ---------------------------------------------------------------- O2 -----------------------
def test_gradient_zero_at_rest_identity():
    sc = scenes.slabs_c1()
    m = build_mesh(sc)
    A = np.tile(np.eye(3).reshape(1, 9), (sc.n_tets, 1))
    p = local_step(m, sc.rest, A)
    g = elastic_gradient(m, sc.rest, p)
    assert np.abs(g).max() < 1e-12 * (m.w.max() / sc.h)


def test_gradient_finite_differences():
    sc = scenes.two_tets()
    m = build_mesh(sc)
    rng = np.random.default_rng(1)
    x = sc.rest + 0.1 * rng.standard_normal(sc.rest.shape)
    A = scenes.random_actuation(sc.n_tets, 0.2, 3)
    p = local_step(m, x, A)
    g = elastic_gradient(m, x, p)
    eps = 1e-6
    fd = np.zeros_like(x)
    for v in range(m.n):
        for a in range(3):
            xp, xm = x.copy(), x.copy()
            xp[v, a] += eps
            xm[v, a] -= eps
            fd[v, a] = (elastic_energy(m, xp, p) - elastic_energy(m, xm, p)) / (2 * eps)
    assert np.abs(g - fd).max() < 1e-7 * np.abs(g).max()


def test_gradient_equals_Hx_minus_rhs():
    sc = scenes.two_tets()
    m = build_mesh(sc)
    rng = np.random.default_rng(2)
    x = sc.rest + 0.05 * rng.standard_normal(sc.rest.shape)
    p = rng.standard_normal((sc.n_tets, 9))
    # rhs = sum_i w_i G_i^T p_i with G_i from the independent formulation
    n = m.n
    rhs = np.zeros(3 * n)
    for i in range(sc.n_tets):
        G = np.zeros((9, 3 * n))
        for k in range(3 * n):
            e = np.zeros(3 * n)
            e[k] = 1.0
            G[:, k] = _F_alt(sc.rest, sc.tets[i:i + 1], e.reshape(n, 3))[0].reshape(9)
        rhs += m.w[i] * G.T @ p[i]
    Hx = np.kron(m.Lap.toarray(), np.eye(3)) @ x.ravel()
    g = elastic_gradient(m, x, p).ravel()
    assert np.abs(g - (Hx - rhs)).max() < 1e-12 * np.abs(rhs).max()
