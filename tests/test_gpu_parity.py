"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same inputs.

Tolerances (north_star): C and S bit-exact as sorted int lists on identical x;
p_i within 1e-5 relative; g-hat 1e-10; dx (lockstep) 1e-8 relative; alpha_m 1e-10 or a logged
discrete flip; positions after N free-running iterations within 1e-5 x bbox diagonal.
"""
import numpy as np
import pytest

import scenes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2312_02999_b200 import pd_ipc
    return pd_ipc


@pytest.fixture(scope="module")
def c1_oracle():
    from oracle import OracleSolver
    sc = scenes.slabs_c1()
    o = OracleSolver(sc)
    log = []
    o.run_frame(sc.rest.copy(), sc.actuation(0), sc.n_iters, log)
    return sc, o, log


def _rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def test_local_step_projections_c1(P):
    from oracle import build_mesh
    from oracle.local import local_step
    sc = scenes.slabs_c1()
    s = P.Solver(sc)
    P.set_debug(s.h, 1)
    rng = np.random.default_rng(3)
    x = sc.rest.copy()
    free = np.setdiff1d(np.arange(sc.n_verts), sc.fixed)
    x[free] += 0.05 * sc.h * rng.standard_normal((free.size, 3))
    P.set_positions(s.h, x)
    s.step(n_iters=1)
    p_gpu = P.get_projections(s.h, sc.n_tets)
    p_ref = local_step(build_mesh(sc), x, sc.actuation(0))
    rel = np.abs(p_gpu - p_ref).max(axis=1) / np.abs(p_ref).max(axis=1)
    assert rel.max() < 1e-5, rel.max()
    assert rel.max() < 1e-11           # expected FP64 agreement
    s.close()


def test_pure_pd_box(P):
    from oracle import OracleSolver
    sc = scenes.box_c5("10k")
    o = OracleSolver(sc)
    s = P.Solver(sc)
    P.set_debug(s.h, 1)
    x = sc.rest.copy()
    for it in range(3):
        ref = o.iterate(x, sc.actuation(0))
        P.set_positions(s.h, x)
        st = s.step(n_iters=1)[0]
        dx = P.get_vector(s.h, sc.n_verts, 1)
        assert _rel(dx, ref["dx"]) < 1e-8
        assert st["alpha"] == 1.0 and st["alpha_max"] == 1.0
        x = ref["x"]
    s.close()


def test_c1_lockstep(P, c1_oracle):
    sc, o, log = c1_oracle
    s = P.Solver(sc)
    P.set_debug(s.h, 1)
    x = sc.rest.copy()
    flips = []
    for k, ref in enumerate(log):
        P.set_positions(s.h, x)
        st = s.step(n_iters=1)[0]
        pt, ee, S = P.get_contacts(s.h)
        rpt = np.stack([ref["C"]["pt"][0], ref["C"]["pt"][1]], 1) if ref["n_pt"] else np.zeros((0, 2))
        ree = np.stack([ref["C"]["ee"][0], ref["C"]["ee"][1]], 1) if ref["n_ee"] else np.zeros((0, 2))
        assert np.array_equal(pt, rpt), f"iteration {k}: PT set differs"
        assert np.array_equal(ee, ree), f"iteration {k}: EE set differs"
        assert np.array_equal(S, ref["S"]), f"iteration {k}: S differs"
        # per-pair barrier gradient and PSD-projected Hessian (<= 1e-9 relative)
        pg, pH = P.get_pair_terms(s.h)
        rg = [ref["pairs"][kd]["h"] for kd in ("pt", "ee") if ref["pairs"].get(kd) is not None]
        rH = [ref["pairs"][kd]["Hp"] for kd in ("pt", "ee") if ref["pairs"].get(kd) is not None]
        if rg:
            rg, rH = np.concatenate(rg), np.concatenate(rH)
            assert pg.shape == rg.shape
            assert _rel(pg, rg) < 1e-9, (k, _rel(pg, rg))
            assert _rel(pH, rH) < 1e-9, (k, _rel(pH, rH))
        g = P.get_vector(s.h, sc.n_verts, 0)
        gref = np.zeros((sc.n_verts, 3))
        gref[o.mesh.free] = ref["ghat"].reshape(-1, 3)
        assert _rel(g, gref) < 1e-10, (k, _rel(g, gref))
        dx = P.get_vector(s.h, sc.n_verts, 1)
        assert _rel(dx, ref["dx"]) < 1e-8, (k, _rel(dx, ref["dx"]))
        if abs(st["alpha_max"] - ref["alpha_m"]) > 1e-10 * ref["alpha_m"]:
            flips.append((k, "alpha_m", st["alpha_max"], ref["alpha_m"]))
        # alpha = alpha_m 2^-h: same halving count, value within alpha_m's tolerance
        if st["ls_trials"] != ref["ls_trials"] or abs(st["alpha"] - ref["alpha"]) > 1e-10 * ref["alpha"]:
            flips.append((k, "alpha", st["alpha"], ref["alpha"]))
        xg = s.positions()
        if not flips:
            assert np.abs(xg - ref["x"]).max() < 1e-9 * sc.bbox_diag()
        x = ref["x"]
    assert len(flips) <= 2, flips
    s.close()


def test_c1_free_running(P, c1_oracle):
    sc, o, log = c1_oracle
    s = P.Solver(sc)
    stats = s.step(n_iters=sc.n_iters)[0]
    xg = s.positions()
    err = np.abs(xg - log[-1]["x"]).max()
    assert err <= 1e-5 * sc.bbox_diag(), err
    assert stats["flags"] == 0
    s.close()


def test_face_small_lockstep(P):
    from oracle import OracleSolver
    sc = scenes.face_small(n_frames=2)
    o = OracleSolver(sc)
    A = sc.actuation(1) * 0 + np.tile(np.eye(3).reshape(1, 9), (sc.n_tets, 1))
    A[:, 4] += 0.5 * sc.meta["lip_mask"]          # full lip actuation at once (App. A.13)
    s = P.Solver(sc, A=A[None])
    P.set_debug(s.h, 1)
    x = sc.rest.copy()
    seen_contact = False
    for k in range(8):
        ref = o.iterate(x, A)
        P.set_positions(s.h, x)
        st = s.step(n_iters=1)[0]
        pt, ee, S = P.get_contacts(s.h)
        assert pt.shape[0] == ref["n_pt"] and ee.shape[0] == ref["n_ee"]
        assert np.array_equal(S, ref["S"])
        seen_contact |= ref["n_pt"] + ref["n_ee"] > 0
        dx = P.get_vector(s.h, sc.n_verts, 1)
        assert _rel(dx, ref["dx"]) < 1e-8, (k, _rel(dx, ref["dx"]))
        x = ref["x"]
    assert seen_contact
    s.close()


def test_c2_full_size_lockstep(P):
    """BASELINE configs[1] at full size (47.5k tets), in the bench's launch configuration: run the
    GPU into the contact regime, then one lockstep iteration against the oracle from the same x."""
    from oracle import OracleSolver
    sc = scenes.face_c2(n_frames=60)
    s = P.Solver(sc)
    for f in range(22):
        s.step(A_next=sc.actuation(f)[None], n_iters=20)
    x = s.positions()
    A = sc.actuation(22)
    o = OracleSolver(sc)
    P.set_debug(s.h, 1)
    for k in range(2):
        ref = o.iterate(x, A)
        P.set_positions(s.h, x)
        st = s.step(A_next=A[None], n_iters=1)[0]
        pt, ee, S = P.get_contacts(s.h)
        assert ref["n_pt"] + ref["n_ee"] > 0, "not in the contact regime"
        assert pt.shape[0] == ref["n_pt"] and ee.shape[0] == ref["n_ee"]
        assert np.array_equal(pt[:, 0], ref["C"]["pt"][0]) and np.array_equal(pt[:, 1], ref["C"]["pt"][1])
        assert np.array_equal(ee[:, 0], ref["C"]["ee"][0]) and np.array_equal(ee[:, 1], ref["C"]["ee"][1])
        assert np.array_equal(S, ref["S"])
        g = P.get_vector(s.h, sc.n_verts, 0)
        gref = np.zeros((sc.n_verts, 3))
        gref[o.mesh.free] = ref["ghat"].reshape(-1, 3)
        assert _rel(g, gref) < 1e-10
        dx = P.get_vector(s.h, sc.n_verts, 1)
        assert _rel(dx, ref["dx"]) < 1e-8, _rel(dx, ref["dx"])
        assert abs(st["alpha_max"] - ref["alpha_m"]) <= 1e-10 * ref["alpha_m"]
        x = ref["x"]
    s.close()


def test_sequences_are_independent_and_deterministic(P):
    """n_seq = 2 with different actuations: each sequence equals its single-sequence run bit for
    bit, and a rerun reproduces it bit for bit (deterministic assembly, no atomics order)."""
    sc = scenes.slabs_c1()
    A1 = sc.actuation(0)
    A2 = A1.copy()
    A2[:, 8] = 1.2                        # a different (symmetric, det > 0) actuation
    both = P.Solver(sc, A=np.stack([A1, A2]), n_seq=2)
    both.step(n_iters=8)
    xs = [both.positions(0), both.positions(1)]
    both.close()
    for A, xb in ((A1, xs[0]), (A2, xs[1])):
        for _ in range(2):
            one = P.Solver(sc, A=A[None])
            one.step(n_iters=8)
            assert np.array_equal(one.positions(), xb)
            one.close()
    assert not np.array_equal(xs[0], xs[1])


def test_degenerate_meshes(P):
    """Edge cases: a single tet and two tets without a collision surface (pure PD, no contact
    work at all) step to the oracle's result."""
    from oracle import OracleSolver
    for sc in (scenes.single_tet(), scenes.two_tets()):
        o = OracleSolver(sc)
        A = np.tile(np.diag([1.2, 1.0, 0.9]).reshape(1, 9), (sc.n_tets, 1))
        s = P.Solver(sc, A=A[None])
        st = s.step(n_iters=1)[0]
        ref = o.iterate(sc.rest.copy(), A)
        assert st["n_S"] == 0 and st["n_active"] == 0
        assert np.abs(s.positions() - ref["x"]).max() <= 1e-9 * max(sc.bbox_diag(), 1e-300)
        s.close()


def test_sigma_reuse_is_exact(P):
    """V_s, K_s and Sigma_s are functions of S and the constant factor only: reusing them while S
    is unchanged must give bit-identical iterates to recomputing them every iteration."""
    sc = scenes.face_small(n_frames=2)
    A = np.tile(np.eye(3).reshape(1, 9), (sc.n_tets, 1))
    A[:, 4] += 0.5 * sc.meta["lip_mask"]
    xs, reused = [], []
    for reuse in (True, False):
        # (the low-rank Sigma_s update, exact only in exact arithmetic, is off here)
        s = P.Solver(sc, A=A[None], sigma_reuse=reuse, debug_flags=P.DBG_NO_SIGMA_UPDATE)
        st = s.step(n_iters=40)[0]
        xs.append(s.positions())
        reused.append(st["sigma_reused"])
        s.close()
    assert np.array_equal(xs[0], xs[1])
    assert reused[0] > 0 and reused[1] == 0, reused


@pytest.mark.parametrize("backend", [2])
def test_sigma_update_tracks_full_sweep(P, backend):
    """When S changes by a few vertices, Sigma_s = K_s^{-1} is updated by low-rank steps (removal:
    Sigma_kk - Sigma_kR Sigma_RR^-1 Sigma_Rk; addition: the bordered inverse with the Schur
    complement of the added block) instead of the full sweep: the iterates must agree with
    sweeping afresh to rounding (updates actually taken)."""
    sc = scenes.face_small(n_frames=2)
    A = np.tile(np.eye(3).reshape(1, 9), (sc.n_tets, 1))
    A[:, 4] += 0.5 * sc.meta["lip_mask"]
    xs, upd = [], []
    for flags in (0, P.DBG_NO_SIGMA_UPDATE):
        s = P.Solver(sc, A=A[None], reduced_backend=backend, debug_flags=flags)
        st = s.step(n_iters=40)[0]
        xs.append(s.positions())
        upd.append(st["sigma_updated"])
        s.close()
    assert upd[0] > 0 and upd[1] == 0, upd
    err = np.abs(xs[0] - xs[1]).max()
    assert err < 1e-9 * sc.bbox_diag(), err


def test_candidate_reuse_is_exact(P):
    """Iterations after the first of a batch take the previous iteration's swept candidate list
    (a superset of the pairs within d_hat at the new positions): the active sets, hence the
    iterates, must be bit-identical to running the static broad phase every iteration."""
    sc = scenes.face_small(n_frames=2)
    A = np.tile(np.eye(3).reshape(1, 9), (sc.n_tets, 1))
    A[:, 4] += 0.5 * sc.meta["lip_mask"]
    xs, nact = [], []
    for reuse in (True, False):
        s = P.Solver(sc, A=A[None], cand_reuse=reuse)
        st = s.step(n_iters=40)[0]
        xs.append(s.positions())
        nact.append(st["n_active"])
        s.close()
    assert nact[0] > 0 and nact[0] == nact[1]
    assert np.array_equal(xs[0], xs[1])
