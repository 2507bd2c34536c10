"""Pins of the oracle's SURVEY 8(f) f3 options (CPU, no GPU): the true-energy line search and
the adaptive barrier stiffness.

True energy (Eq. 1, E_i = min_R ||F_i - R A_i||^2, R = polar(F_i A_i) :79; Z6's 1/2):
  * closed forms: zero on F_i = Q A_i (any rotation Q, uniform A); diag(2, 3, -1) with A = I
    gives 9, not the reflection's 5 (R in SO(3): the reflection fix);
  * an independent library polar factor (scipy.linalg.polar) gives the same per-element values;
  * majorisation: E(y) <= E_p(y) (the surrogate with p fixed at x), equality at y = x;
  * envelope theorem: d/dalpha E(x + alpha dx) at 0 equals g_el . dx (central differences);
  * the line search: at the same alpha dE_true <= dE_surrogate, so alpha_true >= alpha_surrogate.
Adaptive kappa (IPC's rule, reading R-kappa): the rule's cases, and a
C1 run in which kappa doubles exactly where the rule says, with the barrier terms linear in kappa.
"""
import dataclasses

import numpy as np
import pytest

import scenes
from oracle import OracleSolver, build_mesh
from oracle.local import (elastic_energy, elastic_gradient, local_step, true_elastic_energies,
                          true_elastic_energy)
from oracle.solver import kappa_update



def _one_tet_mesh():
    sc = scenes.slabs_c1()
    return build_mesh(sc), sc


def _rot(rng):
    Q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    return Q * np.sign(np.linalg.det(Q))


def test_true_energy_zero_on_rotated_actuated_shape():
    m, sc = _one_tet_mesh()
    A = sc.actuation(0).reshape(-1, 3, 3)
    assert np.allclose(A, A[0])                     # C1: uniform A = diag(1, 1, 1.25)
    Q = _rot(np.random.default_rng(3))
    x = sc.rest @ (Q @ A[0]).T                      # F_i = Q A for every element
    e = true_elastic_energies(m, x, A.reshape(-1, 9))
    assert np.abs(e).max() < 1e-24, np.abs(e).max()


def test_true_energy_reflection_closed_form():
    m, sc = _one_tet_mesh()
    Fd = np.diag([2.0, 3.0, -1.0])
    x = sc.rest @ Fd.T                              # F_i = diag(2, 3, -1): det < 0
    eye = np.tile(np.eye(3).reshape(1, 9), (sc.n_tets, 1))
    e = true_elastic_energies(m, x, eye)
    # min over SO(3) of ||F - R||^2 = |F|^2 + 3 - 2 max tr(R^T F); over the diagonal rotations
    # tr = 4 (I), 0, 2, -6, and I is the SVD route's answer (sigma = 3, 2, 1 with the smallest
    # one's sign flipped): e = 14 + 3 - 8 = 9 (a reflection diag(1, 1, -1) would give 5)
    assert np.allclose(e, 9.0, rtol=0, atol=1e-12), (e.min(), e.max())


def test_true_energy_equals_scipy_polar():
    from scipy.linalg import polar
    sc = scenes.face_small(n_frames=2)
    m = build_mesh(sc)
    rng = np.random.default_rng(5)
    x = sc.rest + 0.1 * sc.h * rng.standard_normal(sc.rest.shape)
    A9 = sc.actuation(1)
    F = m.deformation_gradients(x)
    A = A9.reshape(-1, 3, 3)
    ref = np.empty(sc.n_tets)
    for i in range(sc.n_tets):
        U, _ = polar(F[i] @ A[i])                   # F A = U P, U orthogonal
        assert np.linalg.det(U) > 0                 # no inverted element at this noise level
        ref[i] = np.sum((F[i] - U @ A[i]) ** 2)
    e = true_elastic_energies(m, x, A9)
    assert np.abs(e - ref).max() <= 1e-12 * np.abs(ref).max()


def test_true_energy_majorised_by_surrogate():
    sc = scenes.face_small(n_frames=2)
    m = build_mesh(sc)
    rng = np.random.default_rng(6)
    A9 = sc.actuation(1)
    x = sc.rest + 0.05 * sc.h * rng.standard_normal(sc.rest.shape)
    p = local_step(m, x, A9)
    E0, Ep0 = true_elastic_energy(m, x, A9), elastic_energy(m, x, p)
    assert abs(E0 - Ep0) <= 1e-13 * Ep0
    for k in range(5):
        y = x + 0.05 * sc.h * rng.standard_normal(x.shape)
        assert true_elastic_energy(m, y, A9) <= elastic_energy(m, y, p) * (1 + 1e-14)


def test_true_energy_gradient_is_g_el():
    """Envelope theorem: grad E(x) = sum w G^T (G x - p(x)) (PAPER.md:97 with R at its minimiser)."""
    sc = scenes.face_small(n_frames=2)
    m = build_mesh(sc)
    rng = np.random.default_rng(7)
    A9 = sc.actuation(1)
    x = sc.rest + 0.05 * sc.h * rng.standard_normal(sc.rest.shape)
    dx = sc.h * rng.standard_normal(x.shape)
    g = elastic_gradient(m, x, local_step(m, x, A9))
    h = 1e-5
    fd = (true_elastic_energy(m, x + h * dx, A9) - true_elastic_energy(m, x - h * dx, A9)) / (2 * h)
    an = float(np.sum(g * dx))
    assert abs(fd - an) <= 1e-6 * abs(an), (fd, an)


def test_true_line_search_takes_at_least_the_surrogate_step():
    """dE_true(alpha) <= dE_surrogate(alpha) at every alpha (majorisation), so the halving search
    stops no later: alpha_true >= alpha_surrogate from the same state (stiff C1: halvings)."""
    sc = scenes.slabs_c1()
    sc = dataclasses.replace(sc, kappa=sc.kappa * 1e8)
    A = sc.actuation(0)
    osur = OracleSolver(sc, s_gap=1e-5)
    otru = OracleSolver(sc, s_gap=1e-5, ls_energy="true")
    x = sc.rest.copy()
    halved = 0
    for k in range(6):
        rs, rt = osur.iterate(x, A), otru.iterate(x, A)
        assert np.array_equal(rs["dx"], rt["dx"])
        assert rt["alpha"] >= rs["alpha"], (k, rt["alpha"], rs["alpha"])
        if rs["alpha"] == rt["alpha"] and rs["alpha"] > 0:
            assert rt["dE"] <= rs["dE"] + 1e-12 * abs(rs["dE"])
        halved += rs["ls_trials"] > 1
        x = rs["x"]
    assert halved >= 1


@pytest.mark.parametrize("kappa,d2min,d2prev,eps,kmax,expect", [
    (1.0, 0.25, 0.36, 1.0, 100.0, 2.0),      # below eps and decreasing: doubles
    (1.0, 0.25, 0.25, 1.0, 100.0, 1.0),      # not strictly decreasing
    (1.0, 0.36, 0.25, 1.0, 100.0, 1.0),      # increasing
    (1.0, 1.0, np.inf, 1.0, 100.0, 1.0),     # d = eps is not below eps
    (1.0, 0.99, np.inf, 1.0, 100.0, 2.0),    # first contact below eps
    (60.0, 0.1, 0.2, 1.0, 100.0, 100.0),     # capped at kappa_max
    (1.0, np.inf, np.inf, 1.0, 100.0, 1.0),  # empty C
])
def test_kappa_update_rule(kappa, d2min, d2prev, eps, kmax, expect):
    assert kappa_update(kappa, d2min, d2prev, eps, kmax) == expect


def test_adaptive_kappa_on_c1():
    sc = scenes.slabs_c1()
    eps = sc.d_hat            # every active pair is below d_hat: kappa doubles whenever d_min drops
    o = OracleSolver(sc, kappa_adapt_eps=eps)
    o1 = OracleSolver(sc)
    A = sc.actuation(0)
    x = sc.rest.copy()
    kap, prev, doubled = sc.kappa, np.inf, 0
    for k in range(12):
        r = o.iterate(x, A)
        # the rule re-derived from the logged active distances
        d2 = np.concatenate([r["C"]["pt"][3], r["C"]["ee"][3]])
        dmin = float(d2.min()) if d2.size else np.inf
        if dmin < eps * eps and dmin < prev:
            kap, doubled = min(2 * kap, 100 * sc.kappa), doubled + 1
        prev = dmin
        assert r["kappa"] == kap
        # every barrier term is linear in kappa: the fixed-kappa oracle's terms at the same x scale
        if r["pairs"]:
            r1 = o1.iterate(x, A)
            assert abs(r["EB"] - r1["EB"] * kap / sc.kappa) <= 1e-12 * abs(r["EB"])
        x = r["x"]
    assert doubled >= 2
