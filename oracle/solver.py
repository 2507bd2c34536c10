"""O6, O8, O9 and the Algorithm 1 driver (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

PAPER.md:101-121 (Algorithm 1), one iteration:
  p_i <- GetProjection(x, i)                        (Eq. 1; oracle.local.local_step)
  C <- UpdateConstraintSet(x, d_0)                  (section 2.2; oracle.contact.active_set)
  H-hat <- H + PositiveDefinite(script-B(x, C))     (Eq. 4; per-pair PSD)
  g-hat <- sum_i w_i G_i^T (G_i x - p_i) + grad B   (Eq. 4)
  dx <- -H-hat^{-1} g-hat                           (Eq. 4; O6: the FULL sparse solve -- the
                                                     paper's section 3 reduced solves must equal
                                                     this)
  alpha_m <- CCD(x, dx)                             (oracle.ccd.alpha_max)
  alpha <- LineSearch(x, dx, alpha_m)               (O8; current iterate x, not x_t)
  x <- x + alpha dx                                 (O9)
Options: ls_energy="true" evaluates the line search on the true energy (R
re-minimised per trial); kappa_adapt_eps > 0 adapts kappa per iteration (kappa_update).
Readings: Z6 objective 1/2 sum w E_i + kappa sum b; Z7 line search on the
surrogate with p fixed, dE(alpha) = alpha g_el^T dx + 1/2 alpha^2 sum_a dx_a^T L dx_a
+ kappa sum_{swept}[b(d(alpha)) - b(d(0))]; Z8 strict dE < 0, halving, at most 30 halvings,
then alpha = 0 with a stall flag; Z10 fixed N iterations per frame; Z11 Dirichlet DOFs
eliminated.  The full solve uses scipy's sparse LU (SuperLU) as the library factorisation and
asserts ||H-hat dx + g-hat|| <= 1e-10 ||g-hat||.
"""
from __future__ import annotations

import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import barrier as Bm
from . import ccd as Cc
from . import contact as Ct
from .local import elastic_gradient, local_step, true_elastic_energies
from .setup import build_mesh

STALL = 1


def kappa_update(kappa: float, d2min: float, d2prev: float, eps: float, kappa_max: float) -> float:
    """Adaptive barrier stiffness ("In IPC, kappa is initialized according to the
    average stiffness of the soft body and adaptively adjusted"; the rule is IPC's, which the
    paper does not restate -- DESIGN.md reading R-kappa): kappa doubles, capped at kappa_max,
    when the minimum active-pair distance is below eps AND decreased since the previous
    iteration.  Compared on squared distances (d2min < eps^2, d2min < d2prev); an empty C has
    d2min = +inf (never doubles)."""
    if d2min < eps * eps and d2min < d2prev:
        return min(2.0 * kappa, kappa_max)
    return kappa


class OracleSolver:
    def __init__(self, scene, s_gap=0.1, accd_max_iters=10_000, ls_max_halvings=30, ls_energy="surrogate",
                 kappa_adapt_eps=0.0, kappa_max=None):
        self.scene = scene
        self.mesh = build_mesh(scene)
        self.dh = float(scene.d_hat)
        self.kappa = float(scene.kappa)
        self.s_gap = s_gap
        self.accd_max_iters = accd_max_iters
        self.ls_max_halvings = ls_max_halvings
        assert ls_energy in ("surrogate", "true")
        self.ls_energy = ls_energy                      # surrogate E_p or true E
        self.kappa_adapt_eps = float(kappa_adapt_eps)   # > 0: adaptive kappa (kappa_update)
        self.kappa_max = 100.0 * self.kappa if kappa_max is None else float(kappa_max)
        self.d2prev = np.inf                            # min active d^2 of the previous iteration
        m = self.mesh
        self.free_dof = (3 * m.free[:, None] + np.arange(3)[None, :]).ravel()
        Lff = m.Lap[m.free][:, m.free]
        self.H_free = sp.kron(Lff, sp.identity(3), format="csc")
        self.has_surface = m.tris.shape[0] > 0
        self.timers = dict(ipc=0.0, gstep=0.0, ccd=0.0, ls=0.0, misc=0.0)

    # ------------------------------------------------------------------------------------
    def iterate(self, x: np.ndarray, A9: np.ndarray) -> dict:
        m, dh, kappa = self.mesh, self.dh, self.kappa
        t0 = time.perf_counter()
        p = local_step(m, x, A9)                                  # Alg. 1 :108-110
        g_el = elastic_gradient(m, x, p)                          # (n,3)
        t1 = time.perf_counter()
        self.timers["misc"] += t1 - t0
        if self.has_surface:
            s = m.W @ x
            C = Ct.active_set(s, m.tris, m.edges, dh)             # Alg. 1 :111
            if self.kappa_adapt_eps > 0:                          # f3: adaptive kappa, then every
                d2 = np.concatenate([C["pt"][3], C["ee"][3]])     # use of kappa this iteration
                d2min = float(d2.min()) if d2.size else np.inf
                self.kappa = kappa_update(self.kappa, d2min, self.d2prev, self.kappa_adapt_eps, self.kappa_max)
                self.d2prev = d2min
                kappa = self.kappa
            S = Ct.contact_vertex_set(m.W, m.free_pos, C, m.tris, m.edges)
            gB, HB, EB, pairs = Ct.barrier_derivatives(m, s, C, dh, kappa)
        else:
            s = np.zeros((0, 3))
            C = {k: (np.zeros(0, int),) * 2 + (np.zeros(0, int), np.zeros(0)) for k in ("pt", "ee")}
            S = np.zeros(0, dtype=np.int64)
            gB, HB, EB, pairs = np.zeros((m.n, 3)), None, 0.0, {}
        t2 = time.perf_counter()
        self.timers["ipc"] += t2 - t1
        ghat = (g_el + gB)[m.free].ravel()                        # Alg. 1 :113
        Hhat = self.H_free if HB is None else \
            (self.H_free + HB[self.free_dof][:, self.free_dof]).tocsc()   # Alg. 1 :112
        lu = spla.splu(Hhat)
        dxf = -lu.solve(ghat)                                     # Alg. 1 :114
        res = np.linalg.norm(Hhat @ dxf + ghat)
        assert res <= 1e-10 * max(np.linalg.norm(ghat), 1e-300), ("residual", res)
        dx = np.zeros((m.n, 3))
        dx[m.free] = dxf.reshape(-1, 3)
        t3 = time.perf_counter()
        self.timers["gstep"] += t3 - t2
        if self.has_surface:
            ds = m.W @ dx
            am, sw = Cc.alpha_max(s, ds, m.tris, m.edges, dh, self.s_gap, self.accd_max_iters)
        else:
            ds, am, sw = None, 1.0, None
        t4 = time.perf_counter()
        self.timers["ccd"] += t4 - t3
        alpha, trials, flags, dE = self.line_search(x, s, dx, ds, g_el, sw, am, A9)
        x_new = x + alpha * dx                                    # Alg. 1 :117 (Z1)
        self.timers["ls"] += time.perf_counter() - t4
        return dict(p=p, g_el=g_el, ghat=ghat, s=s, C=C, S=S, pairs=pairs, EB=EB, dx=dx,
                    alpha_m=am, alpha=alpha, ls_trials=trials, flags=flags, dE=dE, x=x_new, kappa=kappa,
                    n_pt=int(C["pt"][0].size), n_ee=int(C["ee"][0].size))

    # ------------------------------------------------------------------------------------
    def line_search(self, x, s, dx, ds, g_el, sw, am, A9=None):
        """O8: halving from alpha_m on the surrogate energy difference; with
        ls_energy == "true" the elastic part is the true energy difference
        E(x + alpha dx) - E(x), E = 1/2 sum_i w_i min_R ||F_i - R A_i||^2 (Eq. 1 re-minimised over
        R at every trial), summed as per-element differences."""
        m, dh, kappa = self.mesh, self.dh, self.kappa
        gTdx = float(np.sum(g_el[m.free] * dx[m.free]))
        quad = float(sum(dx[:, a] @ (m.Lap @ dx[:, a]) for a in range(3)))
        lists = []
        if sw is not None:
            for kind in ("pt", "ee"):
                i0, i1 = sw[kind]
                if i0.size == 0:
                    continue
                ids, Y0 = Ct.pair_points(s, m.tris, m.edges, kind, i0, i1)
                dY = ds[ids].reshape(-1, 12)
                P0 = [Y0[:, 3 * c:3 * c + 3] for c in range(4)]
                b0 = Bm.b(Cc._dist(kind, P0), dh)
                lists.append((kind, P0, [dY[:, 3 * c:3 * c + 3] for c in range(4)], b0))
        if self.ls_energy == "true":
            e0 = true_elastic_energies(m, x, A9)
        alpha = am
        for h in range(self.ls_max_halvings + 1):
            dB = 0.0
            for kind, P0, DY, b0 in lists:
                P = [P0[c] + alpha * DY[c] for c in range(4)]
                dB += float(np.sum(Bm.b(Cc._dist(kind, P), dh) - b0))
            if self.ls_energy == "true":
                dEl = 0.5 * float(np.sum(m.w * (true_elastic_energies(m, x + alpha * dx, A9) - e0)))
            else:
                dEl = alpha * gTdx + 0.5 * alpha * alpha * quad
            dE = dEl + kappa * dB
            if dE < 0.0:
                return alpha, h + 1, 0, dE
            alpha = alpha / 2.0
        return 0.0, self.ls_max_halvings + 1, STALL, 0.0

    # ------------------------------------------------------------------------------------
    def run_until_converged(self, x: np.ndarray, A9: np.ndarray, tol: float, max_iters: int, log=None):
        """Algorithm 1's "while not converged" with SURVEY Z10's optional rule: stop
        after the first iteration whose update moves no vertex by tol or more (max |alpha dx|).
        Returns (x, iterations run)."""
        for k in range(max_iters):
            it = self.iterate(x, A9)
            if log is not None:
                log.append(it)
            x = it["x"]
            if np.abs(it["alpha"] * it["dx"]).max() < tol:
                return x, k + 1
        return x, max_iters

    # ------------------------------------------------------------------------------------
    def run_frame(self, x: np.ndarray, A9: np.ndarray, n_iters: int, log=None):
        """Algorithm 1 for one frame: N fixed iterations from the warm start x (Z10)."""
        for _ in range(n_iters):
            it = self.iterate(x, A9)
            if log is not None:
                log.append(it)
            x = it["x"]
        return x
