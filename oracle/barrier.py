"""O4 barrier terms (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

PAPER.md:88-93 (section 2.2, Eq. 3): B(x) = kappa sum_{k in C} b(d_k(x)), b "logarithm-like",
active for d < d_0.  SURVEY.md Z3/Z4 reading (also SPEC.md:316-317): the IPC barrier in the
UNSQUARED distance, b(d) = -(d - d_hat)^2 ln(d / d_hat) for 0 < d < d_hat, else 0, with
  b'  = -2 (d - d_hat) ln(d/d_hat) - (d - d_hat)^2 / d
  b'' = -2 ln(d/d_hat) - 4 (d - d_hat)/d + (d - d_hat)^2 / d^2.
Per pair: grad d = grad(d^2)/(2d), hess d = (hess(d^2) - 2 grad d grad d^T)/(2d),
h_k = kappa b' grad d, H_k = kappa (b'' grad d grad d^T + b' hess d), and the PSD projection
PositiveDefinite (per pair, 12x12, clamp eigenvalues at 0):
H_k^+ = V max(Lambda, 0) V^T with numpy.linalg.eigh as the library eigensolver.
grad(d^2) and hess(d^2) are obtained by PyTorch CPU autodiff (torch.func) of the type's closed
form, float64 -- an implementation independent of the CUDA path's hand-written derivatives.
"""
from __future__ import annotations

import numpy as np
import torch
from torch.func import grad, hessian, vmap

from . import distance as D


def b(d, dh):
    d = np.asarray(d, dtype=np.float64)
    out = np.zeros_like(d)
    m = (d > 0) & (d < dh)
    dm = d[m]
    out[m] = -(dm - dh) ** 2 * np.log(dm / dh)
    return out


def db(d, dh):
    d = np.asarray(d, dtype=np.float64)
    out = np.zeros_like(d)
    m = (d > 0) & (d < dh)
    dm = d[m]
    out[m] = -2.0 * (dm - dh) * np.log(dm / dh) - (dm - dh) ** 2 / dm
    return out


def d2b(d, dh):
    d = np.asarray(d, dtype=np.float64)
    out = np.zeros_like(d)
    m = (d > 0) & (d < dh)
    dm = d[m]
    out[m] = -2.0 * np.log(dm / dh) - 4.0 * (dm - dh) / dm + (dm - dh) ** 2 / dm ** 2
    return out


# ---- torch closed forms of d^2 over a 12-vector y = (x0, x1, x2, x3) ----------------------
def _t_dot(u, v):
    return u[0] * v[0] + u[1] * v[1] + u[2] * v[2]


def _t_cross(u, v):
    return torch.stack([u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2],
                        u[0] * v[1] - u[1] * v[0]])


def _t_pp(p, q):
    r = p - q
    return _t_dot(r, r)


def _t_pe(p, a, b_):
    c = _t_cross(a - p, b_ - p)
    e = b_ - a
    return _t_dot(c, c) / _t_dot(e, e)


def _t_plane(p, a, b_, c):
    n = _t_cross(b_ - a, c - a)
    t = _t_dot(p - a, n)
    return t * t / _t_dot(n, n)


def _t_ll(a, b_, c, d):
    n = _t_cross(b_ - a, d - c)
    t = _t_dot(c - a, n)
    return t * t / _t_dot(n, n)


def _split(y):
    return y[0:3], y[3:6], y[6:9], y[9:12]


_TYPE_FN = {
    D.PT_A: lambda y: _t_pp(_split(y)[0], _split(y)[1]),
    D.PT_B: lambda y: _t_pp(_split(y)[0], _split(y)[2]),
    D.PT_C: lambda y: _t_pp(_split(y)[0], _split(y)[3]),
    D.PT_AB: lambda y: _t_pe(_split(y)[0], _split(y)[1], _split(y)[2]),
    D.PT_AC: lambda y: _t_pe(_split(y)[0], _split(y)[1], _split(y)[3]),
    D.PT_BC: lambda y: _t_pe(_split(y)[0], _split(y)[2], _split(y)[3]),
    D.PT_FACE: lambda y: _t_plane(*_split(y)),
    D.EE_EE: lambda y: _t_ll(*_split(y)),
    D.EE_PE_A: lambda y: _t_pe(_split(y)[0], _split(y)[2], _split(y)[3]),
    D.EE_PE_B: lambda y: _t_pe(_split(y)[1], _split(y)[2], _split(y)[3]),
    D.EE_PE_C: lambda y: _t_pe(_split(y)[2], _split(y)[0], _split(y)[1]),
    D.EE_PE_D: lambda y: _t_pe(_split(y)[3], _split(y)[0], _split(y)[1]),
    D.EE_PP_AC: lambda y: _t_pp(_split(y)[0], _split(y)[2]),
    D.EE_PP_AD: lambda y: _t_pp(_split(y)[0], _split(y)[3]),
    D.EE_PP_BC: lambda y: _t_pp(_split(y)[1], _split(y)[2]),
    D.EE_PP_BD: lambda y: _t_pp(_split(y)[1], _split(y)[3]),
}


def d2_derivatives(Y: np.ndarray, types: np.ndarray):
    """grad and hessian of the type's d^2 closed form w.r.t. the 12 stacked coordinates."""
    K = Y.shape[0]
    G = np.zeros((K, 12))
    Hs = np.zeros((K, 12, 12))
    for lab, fn in _TYPE_FN.items():
        m = types == lab
        if not m.any():
            continue
        y = torch.from_numpy(np.ascontiguousarray(Y[m])).to(torch.float64)
        G[m] = vmap(grad(fn))(y).numpy()
        Hs[m] = vmap(hessian(fn))(y).numpy()
    return G, Hs


def psd_project(H: np.ndarray) -> np.ndarray:
    """H^+ = V max(Lambda, 0) V^T per 12x12 block (PAPER.md:112 'PositiveDefinite')."""
    lam, V = np.linalg.eigh(H)
    lam = np.maximum(lam, 0.0)
    return np.einsum("kij,kj,klj->kil", V, lam, V)


def pair_terms(Y: np.ndarray, types: np.ndarray, d2: np.ndarray, dh: float, kappa: float):
    """Per active pair: d, b, local gradient h_k (12) and projected Hessian H_k^+ (12x12)."""
    d = np.sqrt(d2)
    G2, H2 = d2_derivatives(Y, types)
    gd = G2 / (2.0 * d)[:, None]
    Hd = (H2 - 2.0 * gd[:, :, None] * gd[:, None, :]) / (2.0 * d)[:, None, None]
    b1 = db(d, dh)
    b2 = d2b(d, dh)
    h = kappa * b1[:, None] * gd
    Hk = kappa * (b2[:, None, None] * gd[:, :, None] * gd[:, None, :] + b1[:, None, None] * Hd)
    Hk = 0.5 * (Hk + Hk.transpose(0, 2, 1))
    return d, b(d, dh), h, psd_project(Hk) if len(Hk) else Hk
