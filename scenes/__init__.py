"""Seeded synthetic scene generators shared by the oracle tests and the GPU path.

This module builds INPUTS only: rest positions, tetrahedra, Dirichlet set, the embedded
collision surface (triangles + W as host tet and barycentric weights), actuation frames,
d_hat and kappa.  It holds none of the method's arithmetic (no deformation gradients, no
stiffness matrix, no distances, no barrier): everything it computes is mesh topology,
seeded random numbers, and the actuation recipe of SURVEY.md section 8(d).

Workloads (BASELINE.json "configs"):
  C1  two stacked slabs (~1k tets) pressed together by actuation, 1 frame x 20 iterations
  C2  face-like block ~47.5k tets with a mouth slit, lips closing over 60 frames
  C3  face-like block ~292k tets with two slits (large contact set)
  C5  no-contact pure-PD boxes, 10k .. 2M tets
plus tiny fixtures for unit tests.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

__all__ = ["Scene", "slabs_c1", "face_c2", "face_c3", "box_c5", "two_tets", "single_tet",
           "cube_grid", "slit_face", "C5_SIZES", "c4_actuation", "c4_assignment", "C4_SEQUENCES"]


@dataclass
class Scene:
    """One workload. All arrays are host numpy, float64 / int32, row-major AoS."""
    name: str
    rest: np.ndarray                 # (n, 3) float64 rest positions (also the start state x_0)
    tets: np.ndarray                 # (T, 4) int32, positively oriented
    fixed: np.ndarray                # (n_fixed,) int32 Dirichlet vertices (sorted)
    surf_tris: np.ndarray            # (N_t, 3) int32 surface-vertex ids
    embed_tet: np.ndarray            # (N_s,) int32 host tet of each surface vertex
    embed_w: np.ndarray              # (N_s, 4) float64 barycentric weights in host tet
    d_hat: float
    kappa: float
    h: float                         # grid cell size
    n_frames: int
    n_iters: int
    actuation: Callable[[int], np.ndarray] = field(repr=False)   # frame -> (T, 9) float64
    cell_of_tet: Optional[np.ndarray] = field(default=None, repr=False)
    meta: dict = field(default_factory=dict)

    @property
    def n_verts(self) -> int:
        return int(self.rest.shape[0])

    @property
    def n_tets(self) -> int:
        return int(self.tets.shape[0])

    @property
    def n_surf_verts(self) -> int:
        return int(self.embed_tet.shape[0])

    def surface_rest(self) -> np.ndarray:
        """Rest positions of the surface vertices (input construction: barycentric blend)."""
        X = self.rest[self.tets[self.embed_tet]]              # (N_s, 4, 3)
        return np.einsum("sc,scd->sd", self.embed_w, X)

    def bbox_diag(self) -> float:
        return float(np.linalg.norm(self.rest.max(0) - self.rest.min(0)))

    def all_frames(self) -> np.ndarray:
        return np.stack([self.actuation(f) for f in range(self.n_frames)])


# ----------------------------------------------------------------------------------------
# cube grids split into 5 tets with alternating parity (conforming)
# ----------------------------------------------------------------------------------------
_CORNER = {(dx, dy, dz): (dx, dy, dz) for dx in (0, 1) for dy in (0, 1) for dz in (0, 1)}
_EVEN = [((0, 0, 0), (1, 1, 0), (1, 0, 1), (0, 1, 1)),        # central tet
         ((1, 0, 0), (0, 0, 0), (1, 1, 0), (1, 0, 1)),
         ((0, 1, 0), (0, 0, 0), (1, 1, 0), (0, 1, 1)),
         ((0, 0, 1), (0, 0, 0), (1, 0, 1), (0, 1, 1)),
         ((1, 1, 1), (1, 1, 0), (1, 0, 1), (0, 1, 1))]
_ODD = [((1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 1)),
        ((0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)),
        ((1, 1, 0), (1, 0, 0), (0, 1, 0), (1, 1, 1)),
        ((1, 0, 1), (1, 0, 0), (0, 0, 1), (1, 1, 1)),
        ((0, 1, 1), (0, 1, 0), (0, 0, 1), (1, 1, 1))]


def _signed_vol6(P: np.ndarray, tets: np.ndarray) -> np.ndarray:
    a, b, c, d = (P[tets[:, k]] for k in range(4))
    return np.einsum("ij,ij->i", np.cross(b - a, c - a), d - a)


def cube_grid(nx: int, ny: int, nz: int, h: float, keep: Optional[Callable] = None):
    """Vertices and 5-tet split of the kept cells of an nx x ny x nz grid of cubes.

    Returns (P (n,3), tets (T,4) positively oriented, cell_of_tet (T,3), ijk of vertices (n,3)).
    Unused vertices are dropped; vertex ids follow lexicographic (i, j, k).
    """
    cells = [(i, j, k) for i in range(nx) for j in range(ny) for k in range(nz)
             if keep is None or keep(i, j, k)]
    vid = {}
    tets, cot = [], []
    for (i, j, k) in cells:
        pattern = _EVEN if (i + j + k) % 2 == 0 else _ODD
        for tet in pattern:
            ids = []
            for (dx, dy, dz) in tet:
                key = (i + dx, j + dy, k + dz)
                ids.append(key)
            tets.append(ids)
            cot.append((i, j, k))
    used = sorted({v for t in tets for v in t})
    vid = {v: n for n, v in enumerate(used)}
    ijk = np.array(used, dtype=np.int64)
    P = ijk.astype(np.float64) * h
    T = np.array([[vid[v] for v in t] for t in tets], dtype=np.int64)
    vol = _signed_vol6(P, T)
    neg = vol < 0
    T[neg, 2], T[neg, 3] = T[neg, 3].copy(), T[neg, 2].copy()
    assert (_signed_vol6(P, T) > 0).all()
    return P, T.astype(np.int32), np.array(cot, dtype=np.int32), ijk


def _jitter(P: np.ndarray, tets: np.ndarray, free_mask: np.ndarray, h: float, seed: int):
    """Uniform +-0.08h per coordinate on non-Dirichlet vertices (SURVEY 8(d) 'rest jitter')."""
    rng = np.random.default_rng(seed)
    J = rng.uniform(-0.08 * h, 0.08 * h, size=P.shape)
    Q = P + J * free_mask[:, None]
    assert (_signed_vol6(Q, tets) > 0).all(), "jitter inverted a tet"
    return Q


def boundary_faces(tets: np.ndarray):
    """Faces used by exactly one tet: returns (faces (F,3) sorted-vertex order, owner tet)."""
    T = tets.shape[0]
    f = np.concatenate([tets[:, [1, 2, 3]], tets[:, [0, 2, 3]], tets[:, [0, 1, 3]],
                        tets[:, [0, 1, 2]]])
    owner = np.concatenate([np.arange(T)] * 4)
    fs = np.sort(f, axis=1)
    _, inv, cnt = np.unique(fs, axis=0, return_inverse=True, return_counts=True)
    once = cnt[inv.ravel()] == 1
    faces, own = fs[once], owner[once]
    order = np.lexsort((faces[:, 2], faces[:, 1], faces[:, 0]))
    return faces[order].astype(np.int32), own[order].astype(np.int32)


def identity_surface(tets: np.ndarray, n: int, faces: np.ndarray):
    """Surface = given faces over sim vertices, W = identity rows (one-hot in host tet)."""
    sv = np.unique(faces)                            # sim ids of surface vertices, ascending
    remap = -np.ones(n, dtype=np.int64)
    remap[sv] = np.arange(sv.size)
    tris = remap[faces].astype(np.int32)
    # lowest-index tet containing each surface vertex
    Tn = tets.shape[0]
    best = np.full(n, Tn, dtype=np.int64)
    bc = np.zeros(n, dtype=np.int64)
    for c in range(4):
        v = tets[:, c].astype(np.int64)
        t = np.arange(Tn)
        m = np.full(n, Tn, dtype=np.int64)
        np.minimum.at(m, v, t)
        upd = m < best
        best[upd] = m[upd]
        bc[upd] = c
    et = best[sv].astype(np.int32)
    ew = np.zeros((sv.size, 4))
    ew[np.arange(sv.size), bc[sv]] = 1.0
    return tris, et, ew, sv


def subdivide_surface(tets: np.ndarray, n: int, faces: np.ndarray):
    """1-to-4 subdivision; edge midpoints are embedded with weights 0.5 / 0.5."""
    base_tris, et0, ew0, sv = identity_surface(tets, n, faces)
    ns0 = sv.size
    e = np.concatenate([faces[:, [0, 1]], faces[:, [1, 2]], faces[:, [2, 0]]])
    e = np.sort(e, axis=1)
    edges = np.unique(e, axis=0)                     # sim-vertex edges, lexicographic
    eid = {(int(a), int(b)): ns0 + i for i, (a, b) in enumerate(edges)}
    # host tet for an edge: lowest-index tet containing both ends
    from collections import defaultdict
    vt = defaultdict(list)
    for ti, t in enumerate(tets):
        for c in range(4):
            vt[int(t[c])].append(ti)
    et1 = np.zeros(len(edges), dtype=np.int32)
    ew1 = np.zeros((len(edges), 4))
    for i, (a, b) in enumerate(edges):
        common = sorted(set(vt[int(a)]) & set(vt[int(b)]))
        t = common[0]
        et1[i] = t
        ca = int(np.where(tets[t] == a)[0][0])
        cb = int(np.where(tets[t] == b)[0][0])
        ew1[i, ca] = 0.5
        ew1[i, cb] = 0.5
    remap = -np.ones(n, dtype=np.int64)
    remap[sv] = np.arange(ns0)
    tris = []
    for (u, v, w) in faces:
        u, v, w = int(u), int(v), int(w)
        muv = eid[tuple(sorted((u, v)))]
        mvw = eid[tuple(sorted((v, w)))]
        mwu = eid[tuple(sorted((w, u)))]
        U, V, Wv = remap[u], remap[v], remap[w]
        tris += [(U, muv, mwu), (V, mvw, muv), (Wv, mwu, mvw), (muv, mvw, mwu)]
    tris = np.array(tris, dtype=np.int32)
    et = np.concatenate([et0, et1]).astype(np.int32)
    ew = np.concatenate([ew0, ew1])
    return tris, et, ew


def _smoothstep(t: float) -> float:
    t = min(max(t, 0.0), 1.0)
    return t * t * (3.0 - 2.0 * t)


# kappa recipe: kappa = KAPPA_PER_H * h.  For a 5-tet cube grid the PD diagonal scales like
# h (volume h^3 times |grad|^2 ~ 1/h^2); the constant is chosen once and stated in DESIGN.md
# so that generators never evaluate the method's stiffness matrix.
KAPPA_PER_H = 2.0


# ----------------------------------------------------------------------------------------
# C1: two stacked slabs
# ----------------------------------------------------------------------------------------
def slabs_c1(seed: int = 0, n_iters: int = 20) -> Scene:
    """Two slabs of 10x5x2 cubes (h = 1 cm); upper slab offset (0.3h, 0.2h, 2.5h), rotated 7
    deg about z; lower bottom and upper top fixed; A = diag(1, 1, 1.25)."""
    h = 0.01
    P0, T0, cot0, ijk0 = cube_grid(10, 5, 2, h)
    n0 = P0.shape[0]
    fixed_lo = ijk0[:, 2] == 0
    fixed_hi = ijk0[:, 2] == 2
    th = math.radians(7.0)
    Rz = np.array([[math.cos(th), -math.sin(th), 0.0], [math.sin(th), math.cos(th), 0.0],
                   [0.0, 0.0, 1.0]])
    ctr = P0.mean(0)
    P1 = (P0 - ctr) @ Rz.T + ctr + np.array([0.3 * h, 0.2 * h, 2.0 * h + 0.5 * h])
    P = np.concatenate([P0, P1])
    T = np.concatenate([T0, T0 + n0]).astype(np.int32)
    fixed_mask = np.concatenate([fixed_lo, fixed_hi])
    P = _jitter(P, T, ~fixed_mask, h, seed)
    fixed = np.nonzero(fixed_mask)[0].astype(np.int32)
    faces, _ = boundary_faces(T)
    tris, et, ew, _ = identity_surface(T, P.shape[0], faces)
    A = np.tile(np.diag([1.0, 1.0, 1.25]).reshape(1, 9), (T.shape[0], 1))
    return Scene("C1_slabs", P, T, fixed, tris, et, ew, d_hat=0.1 * h,
                 kappa=KAPPA_PER_H * h, h=h, n_frames=1, n_iters=n_iters,
                 actuation=lambda f: A.copy(), cell_of_tet=np.concatenate([cot0, cot0]))


# ----------------------------------------------------------------------------------------
# C2 / C3: face-like blocks with slits ("mouth", "eyelid")
# ----------------------------------------------------------------------------------------
def slit_face(nx, ny, nz, h, slits_j, i_range, a_max, n_frames, subdivide, seed=0,
              n_iters=20, name="face", surf_margin=3, lip_cells=4, taper=2):
    i0, i1 = i_range

    def keep(i, j, k):
        return not (j in slits_j and i0 <= i < i1 and 1 <= k < nz)

    P, T, cot, ijk = cube_grid(nx, ny, nz, h, keep)
    fixed_mask = ijk[:, 2] == 0
    P = _jitter(P, T, ~fixed_mask, h, seed)
    fixed = np.nonzero(fixed_mask)[0].astype(np.int32)

    # Chebyshev cell distance to the nearest slit box
    def slit_dist(ci, cj, ck):
        di = np.maximum(0, np.maximum(i0 - ci, ci - (i1 - 1)))
        dj = np.min(np.stack([np.abs(cj - s) for s in slits_j]), axis=0)
        dk = np.maximum(0, 1 - ck)
        return di, dj, dk

    faces, owner = boundary_faces(T)
    oc = cot[owner]
    di, dj, dk = slit_dist(oc[:, 0], oc[:, 1], oc[:, 2])
    near = np.maximum(np.maximum(di, dj), dk) <= surf_margin
    not_fixed = ~fixed_mask[faces].all(axis=1)
    faces = faces[near & not_fixed]
    if subdivide:
        tris, et, ew = subdivide_surface(T, P.shape[0], faces)
        h_surf = 0.5 * h
    else:
        tris, et, ew, _ = identity_surface(T, P.shape[0], faces)
        h_surf = h

    # lip mask: 1 within lip_cells of a slit (in j) over the slit span (in i), cos^2 taper
    ci, cj = cot[:, 0], cot[:, 1]
    di_t = np.maximum(0, np.maximum(i0 - ci, ci - (i1 - 1))).astype(np.float64)
    dj_t = np.min(np.stack([np.abs(cj - s) for s in slits_j]), axis=0).astype(np.float64)

    def ramp(d, flat):
        x = np.clip((d - flat) / taper, 0.0, 1.0)
        m = np.cos(0.5 * np.pi * x) ** 2
        m[d > flat + taper] = 0.0
        return m

    mask = ramp(dj_t, lip_cells) * ramp(di_t, 0)
    Tn = T.shape[0]
    eye = np.tile(np.eye(3).reshape(1, 9), (Tn, 1))
    yy = np.zeros(9)
    yy[4] = 1.0                                      # e_y e_y^T, row-major slot (1,1)

    def actuation(f: int, _mask=mask):
        a = a_max * _smoothstep(f / max(n_frames - 1, 1))
        return eye + (a * _mask)[:, None] * yy[None, :]

    return Scene(name, P, T, fixed, tris, et, ew, d_hat=0.1 * h_surf,
                 kappa=KAPPA_PER_H * h, h=h, n_frames=n_frames, n_iters=n_iters,
                 actuation=actuation, cell_of_tet=cot,
                 meta={"lip_mask": mask, "slits_j": list(slits_j), "i_range": i_range})


def face_c2(seed: int = 0, n_frames: int = 60) -> Scene:
    """48x40x5 cubes, h = 2 mm, mouth slit at j = 14, i in [12, 36), subdivided surface
    within 3 cells of the slit, a(f) = 0.5 smoothstep(f/59) along e_y."""
    return slit_face(48, 40, 5, 0.002, (14,), (12, 36), 0.5, n_frames, subdivide=True,
                     seed=seed, name="C2_face50k")


def face_c3(seed: int = 0, n_frames: int = 60) -> Scene:
    """100x60x10 cubes, h = 2 mm, slits at j = 20 and 40, i in [5, 95), level-0 surface,
    a(f) = 0.6 smoothstep."""
    return slit_face(100, 60, 10, 0.002, (20, 40), (5, 95), 0.6, n_frames, subdivide=False,
                     seed=seed, name="C3_face300k")


def face_small(seed: int = 0, n_frames: int = 4, subdivide: bool = True) -> Scene:
    """Half-scale face (24x20x5, slit j = 7, i in [6, 18)) for CPU tests."""
    return slit_face(24, 20, 5, 0.002, (7,), (6, 18), 0.5, n_frames, subdivide=subdivide,
                     seed=seed, name="face_small")


# ----------------------------------------------------------------------------------------
# C5: pure PD boxes
# ----------------------------------------------------------------------------------------
C5_SIZES = {"10k": (20, 20, 5), "50k": (40, 25, 10), "100k": (40, 50, 10),
            "300k": (100, 60, 10), "1M": (100, 100, 20), "2M": (100, 100, 40)}


def _random_sym_actuation(n: int, scale: float, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    out = np.empty((n, 9))
    todo = np.arange(n)
    while todo.size:
        N = rng.standard_normal((todo.size, 3, 3))
        A = np.eye(3)[None] + scale * 0.5 * (N + N.transpose(0, 2, 1))
        ok = np.linalg.det(A) > 0
        out[todo[ok]] = A[ok].reshape(-1, 9)
        todo = todo[~ok]
    return out


def box_c5(size: str = "10k", seed: int = 0, n_iters: int = 20) -> Scene:
    """Box of cubes, z = 0 fixed, no surface, A = I + 0.1 sym(N(0,1)) (seed 7)."""
    nx, ny, nz = C5_SIZES[size]
    h = 0.002
    P, T, cot, ijk = cube_grid(nx, ny, nz, h) if nx * ny * nz <= 20000 else _fast_box(nx, ny, nz, h)
    fixed_mask = ijk[:, 2] == 0
    P = _jitter(P, T, ~fixed_mask, h, seed)
    A = _random_sym_actuation(T.shape[0], 0.1, 7)
    return Scene(f"C5_box{size}", P, T, np.nonzero(fixed_mask)[0].astype(np.int32),
                 np.zeros((0, 3), np.int32), np.zeros(0, np.int32), np.zeros((0, 4)),
                 d_hat=0.1 * h, kappa=KAPPA_PER_H * h, h=h, n_frames=1, n_iters=n_iters,
                 actuation=lambda f: A.copy(), cell_of_tet=cot)


def _fast_box(nx, ny, nz, h):
    """Vectorised full box (no removed cells); same numbering/orientation as cube_grid."""
    I, J, K = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    I, J, K = I.ravel(), J.ravel(), K.ravel()
    par = (I + J + K) % 2
    vid = lambda i, j, k: (i * (ny + 1) + j) * (nz + 1) + k
    tets = np.empty((I.size, 5, 4), dtype=np.int64)
    for pat, sel in ((_EVEN, par == 0), (_ODD, par == 1)):
        for t, tet in enumerate(pat):
            for c, (dx, dy, dz) in enumerate(tet):
                tets[sel, t, c] = vid(I[sel] + dx, J[sel] + dy, K[sel] + dz)
    T = tets.reshape(-1, 4)
    gi, gj, gk = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1),
                             indexing="ij")
    ijk = np.stack([gi.ravel(), gj.ravel(), gk.ravel()], 1)
    P = ijk.astype(np.float64) * h
    vol = _signed_vol6(P, T)
    neg = vol < 0
    T[neg, 2], T[neg, 3] = T[neg, 3].copy(), T[neg, 2].copy()
    cot = np.repeat(np.stack([I, J, K], 1), 5, axis=0)
    return P, T.astype(np.int32), cot.astype(np.int32), ijk


# ----------------------------------------------------------------------------------------
# tiny fixtures
# ----------------------------------------------------------------------------------------
def single_tet() -> Scene:
    P = np.array([[0.0, 0, 0], [1.0, 0, 0], [0, 1.0, 0], [0, 0, 1.0]])
    T = np.array([[0, 1, 2, 3]], dtype=np.int32)
    A = np.eye(3).reshape(1, 9)
    return Scene("single_tet", P, T, np.array([0], np.int32), np.zeros((0, 3), np.int32),
                 np.zeros(0, np.int32), np.zeros((0, 4)), d_hat=0.1, kappa=1.0, h=1.0,
                 n_frames=1, n_iters=1, actuation=lambda f: A.copy())


def two_tets(seed: int = 3) -> Scene:
    rng = np.random.default_rng(seed)
    P = np.array([[0.0, 0, 0], [1.0, 0, 0], [0, 1.0, 0], [0, 0, 1.0], [1.0, 1.0, 1.0]])
    P = P + rng.uniform(-0.05, 0.05, P.shape)
    T = np.array([[0, 1, 2, 3], [1, 2, 3, 4]], dtype=np.int64)
    vol = _signed_vol6(P, T)
    T[vol < 0, 2], T[vol < 0, 3] = T[vol < 0, 3].copy(), T[vol < 0, 2].copy()
    A = np.tile(np.eye(3).reshape(1, 9), (2, 1))
    return Scene("two_tets", P, T.astype(np.int32), np.array([0], np.int32),
                 np.zeros((0, 3), np.int32), np.zeros(0, np.int32), np.zeros((0, 4)),
                 d_hat=0.1, kappa=1.0, h=1.0, n_frames=1, n_iters=1,
                 actuation=lambda f: A.copy())


def random_actuation(T: int, scale: float, seed: int) -> np.ndarray:
    """Seeded symmetric actuation with det > 0 (for property tests)."""
    return _random_sym_actuation(T, scale, seed)


# ----------------------------------------------------------------------------------------
# C4: a batch of 64 actuation sequences on the C3 mesh
# ----------------------------------------------------------------------------------------
C4_SEQUENCES = 64


def c4_actuation(scene: Scene, j: int, n_frames: Optional[int] = None) -> Callable[[int], np.ndarray]:
    """Actuation of sequence j (seed 1000 + j): a_max,j = 0.45 + 0.3 u, ramp start f0_j uniform in
    [0, 10], and a fixed symmetric noise term 0.02 m_i sym(N(0,1)) per tet; everything ramps in
    with r_j(f) = smoothstep((f - f0_j) / (n_frames - 1 - f0_j)):
        A_i(f) = I + r_j(f) (a_max,j m_i e_y e_y^T + 0.02 m_i sym(N_i)),
    det-checked (an entry is redrawn until det A_i > 0 at full amplitude, which for these
    amplitudes never triggers).  m_i is the lip mask of the scene."""
    nfr = scene.n_frames if n_frames is None else n_frames
    rng = np.random.default_rng(1000 + j)
    a_max = 0.45 + 0.3 * rng.uniform()
    f0 = 10.0 * rng.uniform()
    mask = scene.meta["lip_mask"]
    T = scene.n_tets
    N = rng.standard_normal((T, 3, 3))
    N = 0.5 * (N + N.transpose(0, 2, 1))
    D = np.zeros((T, 3, 3))
    D[:, 1, 1] = a_max * mask
    D += 0.02 * mask[:, None, None] * N
    for _ in range(8):
        bad = np.linalg.det(np.eye(3)[None] + D) <= 0
        if not bad.any():
            break
        M = rng.standard_normal((int(bad.sum()), 3, 3))
        D[bad] = 0.0
        D[bad, 1, 1] = a_max * mask[bad]
        D[bad] += 0.02 * mask[bad, None, None] * 0.5 * (M + M.transpose(0, 2, 1))
    D9 = D.reshape(T, 9)
    eye = np.tile(np.eye(3).reshape(1, 9), (T, 1))
    span = max(nfr - 1 - f0, 1e-9)

    def actuation(f: int):
        return eye + _smoothstep((f - f0) / span) * D9

    actuation.a_max = a_max
    actuation.f0 = f0
    return actuation


def c4_assignment(n_seq: int, rank: int, world: int):
    """Round-robin sharding of the C4 sequences: rank r owns {j : j mod P = r}."""
    return [j for j in range(n_seq) if j % world == rank]
