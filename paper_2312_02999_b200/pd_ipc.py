"""Thin ctypes binding of the C ABI in include/pd_ipc.h (argument marshalling only).

Every step of the PD+IPC iteration runs in the CUDA kernels of libpd_ipc.so; this module only
converts numpy arrays / device pointers to C pointers.  There is no fallback: if the library
is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpd_ipc.so")

E_ARG, E_MESH, E_ACTUATION, E_NOT_SPD, E_INTERSECTING, E_NONFINITE, E_CUDA, E_OOM, E_CAPACITY = \
    -1, -2, -3, -4, -5, -6, -7, -8, -9
FLAG_STALL = 1
DBG_LARGE_SCHUR, DBG_SORT_BROAD, DBG_TINY_HASH, DBG_NO_SIGMA_UPDATE = 1, 2, 4, 8


class pd_ipc_mesh(C.Structure):
    _fields_ = [("n_verts", C.c_int32), ("n_tets", C.c_int32), ("tets", C.POINTER(C.c_int32)),
                ("n_fixed", C.c_int32), ("fixed", C.POINTER(C.c_int32)),
                ("n_surf_verts", C.c_int32), ("n_surf_tris", C.c_int32),
                ("surf_tris", C.POINTER(C.c_int32)), ("embed_tet", C.POINTER(C.c_int32)),
                ("embed_w", C.POINTER(C.c_double))]


class pd_ipc_options(C.Structure):
    _fields_ = [("n_seq", C.c_int32), ("device", C.c_int32), ("ls_max_halvings", C.c_int32),
                ("accd_max_iters", C.c_int32), ("A_on_device", C.c_int32),
                ("max_pairs", C.c_int32), ("accd_s", C.c_double), ("no_sigma_reuse", C.c_int32),
                ("no_cand_reuse", C.c_int32), ("debug_flags", C.c_int32), ("reduced_backend", C.c_int32),
                ("cg_tol", C.c_double), ("cg_max_iters", C.c_int32), ("conv_tol", C.c_double),
                ("ls_energy", C.c_int32), ("kappa_adapt_eps", C.c_double), ("kappa_max", C.c_double)]


class pd_ipc_stats(C.Structure):
    _fields_ = [("iters", C.c_int32), ("n_cand", C.c_int32), ("n_active", C.c_int32),
                ("n_S", C.c_int32), ("ls_trials", C.c_int32), ("flags", C.c_int32),
                ("alpha_max", C.c_double), ("alpha", C.c_double), ("dE", C.c_double),
                ("min_dist", C.c_double), ("ms", C.c_double * 6), ("sigma_reused", C.c_int32),
                ("cg_iters", C.c_int32), ("sigma_updated", C.c_int32), ("kappa", C.c_double)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "ms"}
        d["ms"] = dict(zip(("ipc", "gstep", "ccd", "ls", "misc", "total"), list(self.ms)))
        return d


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() (no CPU fallback exists)")
lib = C.CDLL(LIB_PATH)

_P = C.c_void_p
lib.pd_ipc_create.argtypes = [C.POINTER(pd_ipc_mesh), C.POINTER(C.c_double), C.POINTER(C.c_double),
                              C.c_double, C.c_double, C.POINTER(pd_ipc_options), C.POINTER(_P)]
lib.pd_ipc_create.restype = C.c_int
lib.pd_ipc_step.argtypes = [_P, _P, C.c_int32, C.POINTER(pd_ipc_stats)]
lib.pd_ipc_step.restype = C.c_int
lib.pd_ipc_positions.argtypes = [_P, C.c_int32, C.POINTER(C.c_double)]
lib.pd_ipc_positions.restype = C.c_int
lib.pd_ipc_destroy.argtypes = [_P]
lib.pd_ipc_destroy.restype = None
lib.pd_ipc_last_error.argtypes = [_P]
lib.pd_ipc_last_error.restype = C.c_char_p
lib.pd_ipc_set_positions.argtypes = [_P, C.c_int32, C.POINTER(C.c_double)]
lib.pd_ipc_set_positions.restype = C.c_int
lib.pd_ipc_set_debug.argtypes = [_P, C.c_int32]
lib.pd_ipc_set_debug.restype = C.c_int
lib.pd_ipc_get_projections.argtypes = [_P, C.c_int32, C.POINTER(C.c_double)]
lib.pd_ipc_get_projections.restype = C.c_int
_IP = C.POINTER(C.c_int32)
lib.pd_ipc_get_contacts.argtypes = [_P, C.c_int32, _IP, _IP, _IP, _IP, _IP, _IP]
lib.pd_ipc_get_pair_terms.argtypes = [_P, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double), _IP]
lib.pd_ipc_get_pair_terms.restype = C.c_int
lib.pd_ipc_get_contacts.restype = C.c_int
lib.pd_ipc_get_vector.argtypes = [_P, C.c_int32, C.c_int32, C.POINTER(C.c_double)]
lib.pd_ipc_get_vector.restype = C.c_int
lib.pd_ipc_build_info.argtypes = []
lib.pd_ipc_build_info.restype = C.c_char_p
lib.pd_ipc_debug_factor_solve.argtypes = [C.POINTER(pd_ipc_mesh), C.POINTER(C.c_double),
                                          C.POINTER(C.c_double), C.POINTER(C.c_double),
                                          C.POINTER(C.c_int64)]
lib.pd_ipc_debug_factor_solve.restype = C.c_int
lib.pd_ipc_build_embedding.argtypes = [C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_double), C.c_int32,
                                       C.POINTER(C.c_double), C.c_int32, C.c_double, C.POINTER(C.c_int32),
                                       C.POINTER(C.c_double)]
lib.pd_ipc_build_embedding.restype = C.c_int
lib.pd_ipc_surface_positions.argtypes = [_P, C.c_int32, C.POINTER(C.c_double)]
lib.pd_ipc_surface_positions.restype = C.c_int
lib.pd_ipc_debug_crossings.argtypes = [C.POINTER(pd_ipc_mesh), C.POINTER(C.c_double), C.POINTER(C.c_double)]
lib.pd_ipc_debug_crossings.restype = C.c_int64

lib.pd_ipc_set_timing.argtypes = [_P, C.c_int32]
lib.pd_ipc_set_timing.restype = C.c_int
lib.pd_ipc_kernel_times.argtypes = [_P, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int32]
lib.pd_ipc_kernel_times.restype = C.c_int
lib.pd_ipc_kernel_name.argtypes = [C.c_int32]
lib.pd_ipc_kernel_name.restype = C.c_char_p
lib.pd_ipc_get_info.argtypes = [_P, C.POINTER(C.c_int64), C.c_int32]
lib.pd_ipc_get_info.restype = C.c_int
lib.pd_ipc_launch_count.argtypes = []
lib.pd_ipc_launch_count.restype = C.c_int64

EXPORTED = ["pd_ipc_create", "pd_ipc_step", "pd_ipc_positions", "pd_ipc_destroy",
            "pd_ipc_last_error", "pd_ipc_set_positions", "pd_ipc_set_debug",
            "pd_ipc_get_projections", "pd_ipc_get_contacts", "pd_ipc_get_vector", "pd_ipc_get_pair_terms",
            "pd_ipc_build_info", "pd_ipc_debug_factor_solve", "pd_ipc_debug_crossings",
            "pd_ipc_build_embedding", "pd_ipc_surface_positions", "pd_ipc_set_timing",
            "pd_ipc_kernel_times", "pd_ipc_kernel_name", "pd_ipc_launch_count", "pd_ipc_get_info"]


def set_timing(h, on=True, groups=None):
    """Enable the CUDA-event timers of all kernel groups, or only of `groups` (names)."""
    if groups is not None and on:
        mask = 0
        for g in groups:
            mask |= 1 << [lib.pd_ipc_kernel_name(i).decode() for i in range(32)].index(g)
        _check(lib.pd_ipc_set_timing(h, -mask), h)
        return
    _check(lib.pd_ipc_set_timing(h, int(on)), h)


def kernel_times(h, reset=False):
    """{group name: (ms accumulated, count)} of the timed kernel groups."""
    ms = (C.c_double * 32)()
    cnt = (C.c_int64 * 32)()
    k = lib.pd_ipc_kernel_times(h, ms, cnt, int(reset))
    return {lib.pd_ipc_kernel_name(i).decode(): (ms[i], cnt[i]) for i in range(k)}


INFO_FIELDS = ("n_verts", "n_tets", "n_free", "n_surf_verts", "n_surf_tris", "n_surf_edges", "supernodes",
               "nnz_L", "etree_depth", "capS", "reuse_slots", "n_seq", "bw_row_blocks", "nU", "reduced_backend",
               "region_size", "schur_systems_per_launch")


def get_info(h) -> dict:
    buf = (C.c_int64 * len(INFO_FIELDS))()
    k = lib.pd_ipc_get_info(h, buf, len(INFO_FIELDS))
    if k < 0:
        raise PdIpcError(k, last_error(h))
    return {INFO_FIELDS[i]: int(buf[i]) for i in range(k)}


def launch_count() -> int:
    return int(lib.pd_ipc_launch_count())


class PdIpcError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"pd_ipc error {code}: {msg}")
        self.code = code


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


class _MeshArgs:
    """Keeps the numpy buffers alive while the C struct points at them."""

    def __init__(self, scene):
        self.tets = _i32(scene.tets).reshape(-1, 4)
        self.fixed = _i32(scene.fixed).ravel()
        self.tris = _i32(scene.surf_tris).reshape(-1, 3)
        self.et = _i32(scene.embed_tet).ravel()
        self.ew = _f64(scene.embed_w).reshape(-1, 4)
        self.rest = _f64(scene.rest).reshape(-1, 3)
        self.mesh = pd_ipc_mesh(self.rest.shape[0], self.tets.shape[0], _ip(self.tets),
                                self.fixed.size, _ip(self.fixed), self.et.size, self.tris.shape[0],
                                _ip(self.tris), _ip(self.et), _dp(self.ew))


def last_error(h=None) -> str:
    r = lib.pd_ipc_last_error(h)
    return r.decode() if r else ""


def _check(rc, h=None):
    if rc != 0:
        raise PdIpcError(rc, last_error(h))


def create(scene, A=None, n_seq=1, device=0, A_on_device=False, max_pairs=0,
           ls_max_halvings=30, accd_max_iters=10_000, accd_s=0.1, d_hat=None, kappa=None,
           sigma_reuse=True, cand_reuse=True, debug_flags=0, reduced_backend=0, cg_tol=1e-12,
           cg_max_iters=10000, conv_tol=0.0, ls_energy="surrogate", kappa_adapt_eps=0.0, kappa_max=0.0):
    """pd_ipc_create on a scenes.Scene.  A: (n_seq, T, 9) host actuation (default frame 0)."""
    m = _MeshArgs(scene)
    if A is None:
        A = np.stack([scene.actuation(0)] * n_seq)
    A = _f64(A).reshape(n_seq, -1, 9)
    opt = pd_ipc_options(n_seq, device, ls_max_halvings, accd_max_iters, int(A_on_device),
                         max_pairs, accd_s, 0 if sigma_reuse else 1, 0 if cand_reuse else 1,
                         int(debug_flags), int(reduced_backend), float(cg_tol), int(cg_max_iters),
                         float(conv_tol), {"surrogate": 0, "true": 1}[ls_energy], float(kappa_adapt_eps),
                         float(kappa_max))
    h = _P()
    rc = lib.pd_ipc_create(C.byref(m.mesh), _dp(m.rest), _dp(A),
                           float(scene.d_hat if d_hat is None else d_hat),
                           float(scene.kappa if kappa is None else kappa), C.byref(opt), C.byref(h))
    _check(rc)
    return h


def step(h, A_next=None, n_iters=1, n_seq=1, A_device_ptr=None):
    """pd_ipc_step.  A_next: host (n_seq, T, 9) array, or A_device_ptr: int device address."""
    stats = (pd_ipc_stats * n_seq)()
    if A_device_ptr is not None:
        ptr = _P(int(A_device_ptr))
    elif A_next is not None:
        A_next = _f64(A_next)
        ptr = A_next.ctypes.data_as(_P)
    else:
        ptr = None
    rc = lib.pd_ipc_step(h, ptr, int(n_iters), stats)
    _check(rc, h)
    return [s.as_dict() for s in stats]


def positions(h, n_verts, seq=0):
    out = np.empty((n_verts, 3))
    _check(lib.pd_ipc_positions(h, seq, _dp(out)), h)
    return out


def destroy(h):
    lib.pd_ipc_destroy(h)


def set_positions(h, x, seq=0):
    x = _f64(x)
    _check(lib.pd_ipc_set_positions(h, seq, _dp(x)), h)


def set_debug(h, level=1):
    _check(lib.pd_ipc_set_debug(h, level), h)


def get_projections(h, n_tets, seq=0):
    out = np.empty((n_tets, 9))
    _check(lib.pd_ipc_get_projections(h, seq, _dp(out)), h)
    return out


def get_contacts(h, seq=0):
    n = [C.c_int32(0) for _ in range(3)]
    _check(lib.pd_ipc_get_contacts(h, seq, None, C.byref(n[0]), None, C.byref(n[1]), None,
                                   C.byref(n[2])), h)
    pt = np.empty((n[0].value, 2), np.int32)
    ee = np.empty((n[1].value, 2), np.int32)
    S = np.empty(n[2].value, np.int32)
    _check(lib.pd_ipc_get_contacts(h, seq, _ip(pt), C.byref(n[0]), _ip(ee), C.byref(n[1]),
                                   _ip(S), C.byref(n[2])), h)
    return pt, ee, S


def get_pair_terms(h, seq=0):
    """(grad [n][12], H+ [n][12][12]) of the active pairs of the last iteration (debug >= 1)."""
    n = C.c_int32(0)
    _check(lib.pd_ipc_get_pair_terms(h, seq, None, None, C.byref(n)), h)
    g = np.empty((n.value, 12))
    hp = np.empty((n.value, 78))
    _check(lib.pd_ipc_get_pair_terms(h, seq, _dp(g), _dp(hp), C.byref(n)), h)
    iu = np.triu_indices(12)
    H = np.zeros((n.value, 12, 12))
    H[:, iu[0], iu[1]] = hp
    H[:, iu[1], iu[0]] = hp
    return g, H


def get_vector(h, n_verts, which, seq=0):
    """which: 0 g-hat, 1 dx, 2 elastic gradient -> (n, 3)"""
    out = np.empty((n_verts, 3))
    _check(lib.pd_ipc_get_vector(h, seq, which, _dp(out)), h)
    return out


def build_info() -> str:
    return lib.pd_ipc_build_info().decode()


def debug_factor_solve(scene, b=None):
    """Host-only setup check: factorise L_FF and solve L_FF x = b.  Returns (x, stats)."""
    m = _MeshArgs(scene)
    stats = np.zeros(8, np.int64)
    n = m.rest.shape[0]
    if b is None:
        rc = lib.pd_ipc_debug_factor_solve(C.byref(m.mesh), _dp(m.rest), None, None,
                                           stats.ctypes.data_as(C.POINTER(C.c_int64)))
        _check(rc)
        return None, stats
    b = _f64(b).ravel()
    x = np.empty(n)
    rc = lib.pd_ipc_debug_factor_solve(C.byref(m.mesh), _dp(m.rest), _dp(b), _dp(x),
                                       stats.ctypes.data_as(C.POINTER(C.c_int64)))
    _check(rc)
    return x, stats


def build_embedding(tets, rest, points, tol=1e-9):
    """Host-only: (embed_tet [n_points], embed_w [n_points][4]) of points in the rest tet mesh."""
    tets = _i32(tets).reshape(-1, 4)
    rest = _f64(rest).reshape(-1, 3)
    points = _f64(points).reshape(-1, 3)
    et = np.empty(points.shape[0], np.int32)
    ew = np.empty((points.shape[0], 4))
    rc = lib.pd_ipc_build_embedding(_ip(tets), tets.shape[0], _dp(rest), rest.shape[0], _dp(points),
                                    points.shape[0], float(tol), _ip(et), _dp(ew))
    _check(rc)
    return et, ew


def surface_positions(h, n_surf_verts, seq=0):
    """s = W x of sequence seq, [n_surf_verts][3] (the embedded surface export)."""
    out = np.empty((n_surf_verts, 3))
    _check(lib.pd_ipc_surface_positions(h, seq, _dp(out)), h)
    return out


def debug_crossings(scene, x):
    """Host-only: surface edge-triangle crossings at positions x (n, 3) (the crossing half of
    the intersection-free check of create / set_positions)."""
    m = _MeshArgs(scene)
    x = _f64(x).reshape(-1, 3)
    r = int(lib.pd_ipc_debug_crossings(C.byref(m.mesh), _dp(m.rest), _dp(x)))
    if r < 0:
        raise PdIpcError(r, last_error())
    return r


class Solver:
    """Convenience wrapper: owns a handle for one scene."""

    def __init__(self, scene, **kw):
        self.scene = scene
        self.n_seq = kw.get("n_seq", 1)
        self.h = create(scene, **kw)

    def step(self, A_next=None, n_iters=1, A_device_ptr=None):
        return step(self.h, A_next, n_iters, self.n_seq, A_device_ptr)

    def positions(self, seq=0):
        return positions(self.h, self.scene.n_verts, seq)

    def close(self):
        if self.h:
            destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
