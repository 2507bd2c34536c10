"""Lockstep batching of independent actuation sequences (SURVEY.md 8(e) "per-GPU batching"):
a handle with B sequences runs a1/a2 over (tet, sequence), ONE forward solve with the 3B
gradient right-hand sides, per-sequence contact + Schur steps with their own n_c, and backward
solves of 8 sequences per launch.  Every sequence must equal its single-sequence run BIT FOR BIT
(the batched kernels compute each sequence's columns in the same order as a batch of one), with
one reuse slot per sequence or with shared slots, and the batch must track the oracle.
"""
import os

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


def _run(P, sc, acts, frames, iters, **kw):
    B = len(acts)
    s = P.Solver(sc, A=np.stack([a(0) for a in acts]), n_seq=B, **kw)
    stats = None
    for f in range(frames):
        stats = s.step(A_next=np.stack([a(f) for a in acts]), n_iters=iters)
    xs = [s.positions(b) for b in range(B)]
    s.close()
    return xs, stats


@pytest.mark.parametrize("B", [4, 10])
def test_lockstep_equals_single_runs(P, B):
    sc = scenes.face_small(n_frames=4)
    acts = [scenes.c4_actuation(sc, j, n_frames=4) for j in range(B)]
    xs, stats = _run(P, sc, acts, 4, 10)
    assert max(st["n_S"] for st in stats) > 0          # the batch is in contact
    for j in (0, B - 1, B // 2):
        x1, _ = _run(P, sc, [acts[j]], 4, 10)
        assert np.array_equal(xs[j], x1[0]), j
    # shared reuse slots (memory-limited configuration): still bit-identical
    os.environ["PDIPC_REUSE_SLOTS"] = "1"
    try:
        xs1, _ = _run(P, sc, acts, 4, 10)
    finally:
        del os.environ["PDIPC_REUSE_SLOTS"]
    for j in range(B):
        assert np.array_equal(xs[j], xs1[j]), j
    assert not np.array_equal(xs[0], xs[1])


def test_lockstep_batch_tracks_oracle(P):
    """Three C1 sequences with different actuations in one lockstep handle: each matches the
    oracle's free-running trajectory within 1e-5 x bbox."""
    from oracle import OracleSolver
    sc = scenes.slabs_c1()
    A = sc.actuation(0)
    As = []
    for thick in (1.25, 1.15, 1.3):
        a = A.copy()
        a[:, 8] = thick
        As.append(a)
    s = P.Solver(sc, A=np.stack(As), n_seq=3)
    st = s.step(n_iters=20)
    for b, a in enumerate(As):
        xr = OracleSolver(sc).run_frame(sc.rest.copy(), a, 20)
        assert np.abs(s.positions(b) - xr).max() <= 1e-5 * sc.bbox_diag(), b
        assert st[b]["n_active"] > 0
    s.close()
