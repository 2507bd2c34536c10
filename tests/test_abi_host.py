"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/pd_ipc.h
declares, fails loudly without a GPU, and its host setup (ordering + supernodal Cholesky of
L_FF) solves the oracle's L_FF systems."""
import os
import re

import numpy as np
import pytest

import scenes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def P():
    from paper_2312_02999_b200 import pd_ipc
    return pd_ipc


def test_exports_match_header(P):
    hdr = open(os.path.join(ROOT, "include", "pd_ipc.h")).read()
    declared = set(re.findall(r"\b(pd_ipc_\w+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(P.lib, name), f"{name} declared in pd_ipc.h but not exported"
    assert declared == set(P.EXPORTED)


def test_product_has_no_oracle_dependency():
    """The product path never imports the oracle (the oracle is test infrastructure)."""
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2312_02999_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", src).lower().replace(
                    "the oracle", ""), f"{f} mentions the oracle in code"


def test_create_without_gpu_fails_loudly(P):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.PdIpcError) as e:
        P.create(scenes.slabs_c1())
    assert e.value.code == P.E_CUDA


@pytest.mark.parametrize("kw", [dict(reduced_backend=5), dict(reduced_backend=-1), dict(kappa_adapt_eps=-1.0)])
def test_create_rejects_bad_options(P, kw):
    """Option validation happens before any device work (include/pd_ipc.h: E_ARG)."""
    with pytest.raises(P.PdIpcError) as e:
        P.create(scenes.slabs_c1(), **kw)
    assert e.value.code == P.E_ARG


def test_create_rejects_bad_ls_energy(P):
    opt = P.pd_ipc_options()
    opt.n_seq, opt.ls_energy = 1, 2
    m = P._MeshArgs(scenes.slabs_c1())
    A = P._f64(scenes.slabs_c1().actuation(0))
    h = P._P()
    rc = P.lib.pd_ipc_create(P.C.byref(m.mesh), P._dp(m.rest), P._dp(A), 1e-3, 1.0, P.C.byref(opt), P.C.byref(h))
    assert rc == P.E_ARG


@pytest.mark.parametrize("make", [scenes.slabs_c1, scenes.face_small, lambda: scenes.box_c5("10k")])
def test_host_factor_solves_oracle_laplacian(P, make):
    from oracle import build_mesh
    sc = make()
    m = build_mesh(sc)
    b = np.random.default_rng(1).standard_normal(sc.n_verts)
    x, st = P.debug_factor_solve(sc, b)
    Lff = m.Lap[m.free][:, m.free]
    r = Lff @ x[m.free] - b[m.free]
    assert np.abs(r).max() < 1e-11 * np.abs(b).max()
    assert np.all(x[m.fixed] == 0)
    nsn, nnz, wmax, depth = st[:4]
    assert 0 < nsn <= m.n_free and wmax <= 128 and depth >= 1
    assert nnz >= m.n_free


def test_setup_rejects_bad_input(P):
    sc = scenes.slabs_c1()
    bad = scenes.Scene(**{**sc.__dict__})
    bad.fixed = np.zeros(0, np.int32)
    with pytest.raises(P.PdIpcError) as e:
        P.debug_factor_solve(bad)
    assert e.value.code == P.E_NOT_SPD
    bad = scenes.Scene(**{**sc.__dict__})
    bad.tets = sc.tets.copy()
    bad.tets[0, [2, 3]] = bad.tets[0, [3, 2]]
    with pytest.raises(P.PdIpcError) as e:
        P.debug_factor_solve(bad)
    assert e.value.code == P.E_MESH
    bad = scenes.Scene(**{**sc.__dict__})
    bad.embed_w = sc.embed_w * 0.9
    with pytest.raises(P.PdIpcError) as e:
        P.debug_factor_solve(bad)
    assert e.value.code == P.E_MESH


def test_host_crossing_check_matches_brute_force(P):
    """The crossing half of the create / set_positions intersection check (SURVEY 8(b)
    E_INTERSECTING) counts exactly the edge-triangle piercings of an independent brute-force
    Moller-Trumbore test, on the rest state (none) and on interpenetrating C1 states."""
    from test_oracle_solve import edge_triangle_crossings
    from oracle import build_mesh
    sc = scenes.slabs_c1()
    m = build_mesh(sc)
    assert P.debug_crossings(sc, sc.rest) == 0
    rng = np.random.default_rng(3)
    upper = sc.rest[:, 2] > 2.25 * sc.h
    for shift in (0.8, 1.0, 1.7):
        x = sc.rest.copy()
        x[upper, 2] -= shift * sc.h
        x[upper] += rng.uniform(-0.05, 0.05, (int(upper.sum()), 3)) * sc.h
        ref = edge_triangle_crossings(m.W @ x, m.tris, m.edges)
        assert ref > 0
        assert P.debug_crossings(sc, x) == ref


def test_struct_layouts_match_header(P, tmp_path):
    """The ctypes mirrors of pd_ipc_options / pd_ipc_stats / pd_ipc_mesh have the header's
    size and field offsets (gcc compiles include/pd_ipc.h and prints them)."""
    import ctypes
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    structs = {"pd_ipc_options": P.pd_ipc_options, "pd_ipc_stats": P.pd_ipc_stats, "pd_ipc_mesh": P.pd_ipc_mesh}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "pd_ipc.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'printf("{name} size %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{name} {f} %zu\\n", offsetof({name}, {f}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(root, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for name, cls in structs.items():
        assert got[(name, "size")] == ctypes.sizeof(cls), name
        for f, _ in cls._fields_:
            assert got[(name, f)] == getattr(cls, f).offset, (name, f)
