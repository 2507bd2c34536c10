"""O1 local step and O2 elastic gradient (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

PAPER.md:73-79 (Eq. 1, section 2.1): E_i(x) = min_{R in SO(3)} ||F_i(x) - R A_i||_F^2 =
||G_i x - p_i||^2; "we find the best rotation R_i using the polar decomposition of F_i A_i".
SURVEY.md 8(c) O1 / SPEC.md:114,136: SVD M = U S V^T (numpy LAPACK, s1 >= s2 >= s3 >= 0);
if det(U V^T) < 0 negate U's third column; R = U V^T; p_i = vec_rowmajor(R A_i).

PAPER.md:97, :113 (Eq. 4): the elastic part of g-hat is sum_i w_i G_i^T (G_i x - p_i);
per vertex v that is sum_{i contains v} w_i (F_i - P_i) g_{i,c(v)}.
"""
from __future__ import annotations

import numpy as np


def polar_rotation(M: np.ndarray) -> np.ndarray:
    """Rotation factor of M (..., 3, 3) via SVD with the reflection fix."""
    U, S, Vt = np.linalg.svd(M)
    d = np.linalg.det(U @ Vt)
    U = U.copy()
    U[d < 0, :, 2] *= -1.0
    return U @ Vt


def local_step(mesh, x: np.ndarray, A9: np.ndarray) -> np.ndarray:
    """p_i = vec(R_i A_i), R_i = polar(F_i A_i)  -> (T, 9) row-major (Alg. 1 :108-110)."""
    F = mesh.deformation_gradients(x)
    A = A9.reshape(-1, 3, 3)
    R = polar_rotation(F @ A)
    return (R @ A).reshape(-1, 9)


def elastic_energy(mesh, x: np.ndarray, p: np.ndarray) -> float:
    """Surrogate elastic energy 1/2 sum_i w_i ||G_i x - p_i||^2 (SURVEY Z6/Z7 reading)."""
    F = mesh.deformation_gradients(x).reshape(-1, 9)
    r = F - p
    return 0.5 * float(np.sum(mesh.w * np.einsum("ti,ti->t", r, r)))


def true_elastic_energies(mesh, x: np.ndarray, A9: np.ndarray) -> np.ndarray:
    """Per-element true energies e_i(x) = min_{R in SO(3)} ||F_i(x) - R A_i||_F^2 (Eq. 1,
    PAPER.md:75), the minimiser being the polar rotation of F_i A_i -> (T,).
    Used by the true-energy line search (reading Z7's alternative)."""
    F = mesh.deformation_gradients(x)
    A = A9.reshape(-1, 3, 3)
    R = polar_rotation(F @ A)
    r = (F - R @ A).reshape(-1, 9)
    return np.einsum("ti,ti->t", r, r)


def true_elastic_energy(mesh, x: np.ndarray, A9: np.ndarray) -> float:
    """E(x) = 1/2 sum_i w_i e_i(x) (Eq. 1 with the Z6 factor 1/2)."""
    return 0.5 * float(np.sum(mesh.w * true_elastic_energies(mesh, x, A9)))


def elastic_gradient(mesh, x: np.ndarray, p: np.ndarray) -> np.ndarray:
    """g_el[v] = sum_{i contains v} w_i (F_i - P_i) g_{i,c(v)} on ALL vertices -> (n, 3).

    The free rows of this are Eq. 4's sum_i w_i G_i^T (G_i x - p_i); callers take [free].
    """
    F = mesh.deformation_gradients(x)
    Rm = (F - p.reshape(-1, 3, 3)) * mesh.w[:, None, None]     # w_i (F_i - P_i)
    contrib = np.einsum("tab,tcb->tca", Rm, mesh.g)           # (T,4,3): w (F-P) g_c
    gv = np.zeros((mesh.n, 3))
    np.add.at(gv, mesh.tets.reshape(-1), contrib.reshape(-1, 3))
    return gv
