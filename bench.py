#!/usr/bin/env python
"""Benchmark of the PD+IPC iteration (arXiv 2312.02999) on B200: prints ONE JSON line.

Headline workload (BASELINE.json configs[3]): the batch of 64 seeded
actuation sequences on the ~300k-tet two-slit face mesh (C3), sharded round-robin over the P
GPUs (rank r owns sequences j = r mod P).  Each rank runs its sequences in LOCKSTEP in one
handle.  A bench "step" is one pass of the whole hot path (local step, gather, broad/narrow
phase, contact assembly, contact-reduced global solve, CCD, line search, update) over the rank's
batch, i.e. one PD+IPC iteration of every sequence it owns; 20 steps = one frame.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Per sequence j: untimed preparation = PREP_ITERS iterations from rest under the frame-(F-1)
actuation (the frame-(F-1) equilibrium), then W warm-up steps continuing that frame, then the
K timed steps under the frame-F actuation (F = TIMED_FRAME), warm-started.  The frame subset and
the per-sequence inputs are identical for every P.  value = all ranks' sequence-iterations /
max-over-ranks device time (weak scaling over sequences, no data-path collective); NCCL
all-gathers the per-rank times, statistics and per-sequence position checksums.

Extra fields: C3 single sequence (configs[2]), C2 (configs[1]) and the C5 1M-tet pure-PD
local-step / gather HBM roofline (configs[4]).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ITERS_PER_FRAME = 20
N_SEQ = 64                 # C4 batch
TIMED_FRAME = 30           # F: every sequence is ramped and in contact by frame 30
PREP_ITERS = 20            # untimed iterations from rest under the frame-(F-1) actuation
E2E_STEPS = 10             # end-to-end steps (same handle, continuing frame F)
C2_FRAMES = 60
C2_CONTACT_START = 20


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--seqs", type=int, default=N_SEQ, help="C4 batch size (64 = BASELINE configs[3])")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the C3-single / C2 / C5 fields")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--ref-seconds", type=float, default=150.0)
    ap.add_argument("--c5", default="1M", help="pure-PD box size for the local-step HBM field ('' to skip)")
    return ap.parse_args()


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def _sm_max_mhz():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["sm_max_mhz"])
    except Exception:
        return 1965.0


# ------------------------------------------------------------------------------ clocks -----
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def _host_info():
    model = ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "lscpu_model": model}


# ------------------------------------------------------------------------------ host logic -
def gather_rank_values(vals, world, device):
    """All ranks' per-rank measurements as a (world, len(vals)) array (NCCL on the GPU path; any
    backend works).  The job's time is the max over ranks of the device-timed region."""
    import torch
    import torch.distributed as dist
    mine = torch.tensor(vals, dtype=torch.float64, device=device)
    if world > 1:
        allv = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allv, mine)
        return torch.stack(allv).cpu().numpy()
    return mine.cpu().numpy()[None]


def job_throughput(per_rank_ms, units_per_rank):
    """Whole-job throughput: every rank processed units_per_rank[r] sequence-iterations (weak
    scaling over sequences); the job took the slowest rank's time."""
    return float(sum(units_per_rank)) / (max(per_rank_ms) / 1000.0)


def seq_checksum(x):
    """64-bit checksum of a sequence's positions (float64 bytes), for the cross-P determinism check."""
    import numpy as np
    return int.from_bytes(hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).digest()[:7], "little")


def gather_checksums(pairs, world, device, n_seq):
    """{sequence j: checksum} over all ranks (all_gather of a dense [n_seq] vector, 0 = not mine)."""
    import torch
    import torch.distributed as dist
    v = torch.zeros(n_seq, dtype=torch.int64, device=device)
    for j, c in pairs:
        v[j] = c
    if world > 1:
        allv = [torch.zeros_like(v) for _ in range(world)]
        dist.all_gather(allv, v)
        v = torch.stack(allv).sum(0)
    return {j: int(c) for j, c in enumerate(v.cpu().tolist())}


def combined_checksum(by_seq):
    """One hex digest over all sequences in j order: equal across P iff every trajectory is."""
    h = hashlib.sha256()
    for j in sorted(by_seq):
        h.update(int(by_seq[j]).to_bytes(8, "little"))
    return h.hexdigest()[:16]


# ------------------------------------------------------------------------------ oracle -----
_CPU_SCRIPT = r"""
import json, sys, time
import numpy as np
sys.path.insert(0, sys.argv[1])
import scenes
from oracle import OracleSolver
sc = scenes.face_c3()
j = int(sys.argv[2]); frame = int(sys.argv[3]); budget = float(sys.argv[4])
o = OracleSolver(sc)
A = scenes.c4_actuation(sc, j)(frame)
x = o.iterate(sc.rest.copy(), A)["x"]          # untimed warm-up iteration from rest (no contact yet)
for k in o.timers: o.timers[k] = 0.0
t0 = time.perf_counter(); n = 0
while True:
    it = o.iterate(x, A); x = it["x"]; n += 1
    if time.perf_counter() - t0 >= budget: break
dt = time.perf_counter() - t0
print(json.dumps({"iters": n, "seconds": dt, "n_active": it["n_pt"] + it["n_ee"], "n_S": int(it["S"].size),
                  "timers": o.timers}))
"""


def start_cpu_baseline(j, frame, budget):
    """The oracle as it stands, single thread, on a bounded sample of the same workload, started
    in the background (it needs no GPU): C4 sequence j under its frame-(F-1) actuation from rest,
    one untimed warm-up iteration, then whole timed iterations until the budget is used (at least
    one; an iteration with contact refactorises the full 180k-DOF H-hat)."""
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1",
               NUMEXPR_NUM_THREADS="1", CUDA_VISIBLE_DEVICES="")
    td = tempfile.mkdtemp()
    sp = os.path.join(td, "cpu.py")
    with open(sp, "w") as f:
        f.write(_CPU_SCRIPT)
    return subprocess.Popen([sys.executable, sp, ROOT, str(j), str(frame), str(budget)], env=env,
                            stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)


def finish_cpu_baseline(proc, j, frame, timeout=1200):
    try:
        out, err = proc.communicate(timeout=timeout)
    except subprocess.TimeoutExpired:
        proc.kill()
        out, err = proc.communicate()
    hi = _host_info()
    if proc.returncode != 0 or not out.strip():
        return {"value": None, "unit": "iters/s", "cores": 1, "kind": "oracle", **hi,
                "sample": "failed: " + ((err or "").strip().splitlines() or ["?"])[-1][:200]}
    d = json.loads(out.strip().splitlines()[-1])
    return {"value": d["iters"] / d["seconds"], "unit": "iters/s", "cores": 1, "kind": "oracle", **hi,
            "threads_used": 1,
            "sample": f"{d['iters']} timed oracle iteration(s) of C4 sequence {j} under its frame-{frame} "
                      f"actuation, after one untimed iteration from rest ({d['seconds']:.1f} s, |C| "
                      f"{d['n_active']}, n_c {d['n_S']}); full sparse LU of H-hat per iteration, 1 thread, "
                      f"run concurrently with the GPU measurement on its own host core",
            "stage_s": {k: round(v, 2) for k, v in d["timers"].items()}}


# ------------------------------------------------------------------------------ reference --
def run_reference(a):
    """--impl reference: the CPU oracle as it stands, on this arm's config (C4) and metric.

    A step of the oracle is one iteration of one C4 sequence (the batch's sequences are
    independent, so the rate per sequence-iteration is the batch rate).  One oracle iteration at
    this size refactorises the full 180k-DOF H-hat (tens of seconds), so the run is bounded in
    time: at most min(W, 1) warm-up and K timed iterations, stopping after --ref-seconds; the
    line states the counts actually run."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import scenes
    from oracle import OracleSolver
    sc = scenes.face_c3()
    j = 0
    act = scenes.c4_actuation(sc, j)
    o = OracleSolver(sc)
    x = sc.rest.copy()
    t_all = time.perf_counter()
    w_done = 0
    for _ in range(min(a.warmup, 1)):
        x = o.iterate(x, act(TIMED_FRAME - 1))["x"]
        w_done += 1
    A = act(TIMED_FRAME)
    t0 = time.perf_counter()
    n = 0
    it = None
    while n < a.steps:
        it = o.iterate(x, A)
        x = it["x"]
        n += 1
        if time.perf_counter() - t_all >= a.ref_seconds:
            break
    dt = time.perf_counter() - t0
    v = n / dt
    hi = _host_info()
    line = {"impl": "reference", "metric": "PD+IPC iterations/s", "value": v, "unit": "iters/s",
            "n_gpus": a.gpus, "steps": n, "warmup": w_done, "steps_requested": a.steps,
            "warmup_requested": a.warmup, "ms_per_step": 1000 * dt / n,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, SURVEY.md 8(d) C4)", "frames_per_sec": v / ITERS_PER_FRAME,
            "config": {"workload": "C4: 64 actuation sequences on the ~300k-tet two-slit face (C3 mesh) "
                                   "(BASELINE.json configs[3])",
                       "step": "one oracle PD+IPC iteration of one sequence (bounded sample)",
                       "sample": f"sequence {j}: {w_done} warm-up iteration(s) from rest under the frame-"
                                 f"{TIMED_FRAME - 1} actuation, then {n} timed iteration(s) under frame "
                                 f"{TIMED_FRAME} (time-bounded at {a.ref_seconds:.0f} s)"},
            "cpu_baseline": {"value": v, "unit": "iters/s", "cores": 1, "kind": "oracle", **hi,
                             "sample": f"{n} oracle iteration(s) (|C| {it['n_pt'] + it['n_ee']}, "
                                       f"n_c {int(it['S'].size)})"},
            "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ rooflines --
# FP64 tensor (DMMA, mma.sync.m8n8k4.f64) throughput measured on this pool's B200 over the whole
# GPU by tools/micro/dmma_gpu_peak.cu: 37.12 TFLOP/s at 1965 MHz = 127.6 flop/clk/SM
# (profiles/fp64_gpu_peak_r02.txt; the one-SM figure of tools/micro/fp64_peaks.cu is 128).
# tcgen05 has no f64 kind, so this is the FP64 contraction peak; scaled by the max SM clock.
# cuBLAS DGEMM (torch.matmul float64, 8192^3) reaches 35.45 TFLOP/s on the same GPU: the
# library reference the dense Schur kernel is also quoted against.
DMMA_TFLOPS_MEASURED, DMMA_MEASURED_MHZ = 37.12, 1965.0
DGEMM_CUBLAS_TFLOPS = 35.45
N_SM = 148


def _traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full summary, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
    except Exception:
        return None
    for name, v in t.items():          # template instances are listed as e.g. k_local_step<4>
        if name == kernel or name.startswith(kernel + "<"):
            return v
    return None


def _fp64_peak(sm_max_mhz):
    return DMMA_TFLOPS_MEASURED * sm_max_mhz / DMMA_MEASURED_MHZ


def _ns_steps(floor=1e-10):
    """Steps of the scaled Newton-Schulz sign schedule of k_pair_derivs (k_contact.cu
    contact_init: a = sqrt(3 / (1 + l + l^2)), l <- a l (3 - a^2 l^2) / 2 from l = floor until
    1 - l < 1e-16)."""
    import math
    l, k = floor, 0
    while k < 64:
        a = math.sqrt(3.0 / (1.0 + l + l * l))
        k += 1
        l = 0.5 * a * l * (3.0 - a * a * l * l)
        if 1.0 - l < 1e-16:
            break
    return k


# DMMA flops one sign step issues per pair: two 16x16 (zero-padded 12x12) products with k = 12,
# 4 output tiles x 3 k-steps x 512 flops each
NS_FLOPS_PER_STEP = 2 * 4 * 3 * 512


def rooflines(kt, info, nb, nS_list, reuse_frac, hbm, sm_max_mhz, peak_src, upd_frac=0.0, nA_list=None):
    """Per kernel group: achieved = ALGORITHMIC bytes (flops) per launch / average launch time
    (live CUDA events), DESIGN.md section 5.  kt: {group: (ms, launches)}; nb sequences per
    lockstep iteration; nS_list: n_c of every sequence."""
    out = {}
    T, n, nf, nnzL = info["n_tets"], info["n_verts"], info["n_free"], info["nnz_L"]

    def avg(k):
        ms, c = kt.get(k, (0.0, 0))
        return (ms / c / 1000.0, c) if c else (None, 0)

    t, _ = avg("local_step")
    if t:   # per tet: ids 16 + B 72 + w 8 once; per (tet, seq): A 48 + forces 96; x 32 per vertex and seq
        b = T * (16 + 72 + 8) + nb * (T * (48 + 96) + n * 32)
        out["local_step"] = {"bound": "hbm", "achieved": b / t / 1e9, "peak": hbm, "unit": "GB/s",
                             "frac": b / t / 1e9 / hbm, "bytes_per_launch": b, "avg_launch_us": t * 1e6}
    t, _ = avg("gather")
    if t:
        b = nb * (nf * (8 + 32) + 4 * T * (4 + 24))
        out["gather"] = {"bound": "hbm", "achieved": b / t / 1e9, "peak": hbm, "unit": "GB/s",
                         "frac": b / t / 1e9 / hbm, "bytes_per_launch": b, "avg_launch_us": t * 1e6}
    t, _ = avg("w_el_forward")
    if t:   # the factor (Q blocks, nnz(L) doubles) read once + 3 nb right-hand sides in / out
        b = nnzL * 8 + nb * nf * 32 * 2
        out["w_el_forward"] = {"bound": "hbm", "achieved": b / t / 1e9, "peak": hbm, "unit": "GB/s",
                               "frac": b / t / 1e9 / hbm, "bytes_per_launch": b, "avg_launch_us": t * 1e6,
                               "note": "one launch solves all nb sequences' gradients; dependency-depth bound"}
    t, _ = avg("backward_solve")
    if t:   # ONE launch per iteration for all nb sequences (column tiles of 8 sequences): the factor
        # (nnz(L) doubles) counted once -- the tiles' re-reads of a Q block come from L2 -- plus the
        # right-hand sides in and out
        b = nnzL * 8 + nb * nf * 32 * 2
        out["backward_solve"] = {"bound": "hbm", "achieved": b / t / 1e9, "peak": hbm, "unit": "GB/s",
                                 "frac": b / t / 1e9 / hbm, "bytes_per_iteration": b, "avg_iteration_us": t * 1e6,
                                 "launches_per_iteration": 1, "column_tiles": (nb + 7) // 8}
    t, _ = avg("dense_schur")
    if t and nS_list:
        # per sequence at n_c, m = 3 n_c: Cholesky of the augmented Sigma-hat (m^3 / 3), Sigma_s =
        # K_s^-1 by the full sweep (n_c^3) for the iterations that neither reused it (S unchanged)
        # nor updated it by low-rank steps (counted as 0 flops: conservative), back substitution
        # and t = B u, Z (4 m^2)
        fl = [max(0.0, 1.0 - reuse_frac - upd_frac) * nc ** 3 + (3 * nc) ** 3 / 3.0 + 4 * (3 * nc) ** 2
              for nc in nS_list]
        f = statistics.mean(fl) * info.get("schur_systems_per_launch", 1)   # systems per launch
        pk = _fp64_peak(sm_max_mhz)
        out["dense_schur"] = {"kernel": "k_schur_coop", "bound": "tensor", "achieved": f / t / 1e12, "peak": pk,
                              "unit": "TFLOP/s", "frac": f / t / 1e12 / pk, "flops_per_launch": f,
                              "avg_launch_us": t * 1e6, "n_c_mean": statistics.mean(nS_list),
                              "systems_per_launch": info.get("schur_systems_per_launch", 1),
                              "frac_of_cublas_dgemm": f / t / 1e12 / DGEMM_CUBLAS_TFLOPS,
                              "peak_source": "FP64 DMMA measured over the whole GPU (tools/micro/dmma_gpu_peak.cu, "
                                             "profiles/fp64_gpu_peak_r02.txt), scaled to the max SM clock"}
    t, c = avg("pair_derivatives")
    if t and nA_list:
        # warp per active pair; the PSD projection's sign iteration dominates: issued DMMA flops
        # (padded 16x16 tiles) of the fixed schedule per pair, per sequence's launch
        f = statistics.mean(nA_list) * _ns_steps() * NS_FLOPS_PER_STEP
        pk = _fp64_peak(sm_max_mhz)
        out["pair_derivatives"] = {"bound": "tensor", "achieved": f / t / 1e12, "peak": pk, "unit": "TFLOP/s",
                                   "frac": f / t / 1e12 / pk, "flops_per_launch": f, "avg_launch_us": t * 1e6,
                                   "launches": c, "n_active_mean": statistics.mean(nA_list),
                                   "note": "issued DMMA flops of the Newton-Schulz sign iteration (%d steps, "
                                           "zero-padded 16x16 tiles); the timed group also holds the clears "
                                           "of a5-a6" % _ns_steps()}
    for k in ("panel_forward", "contact_assembly", "narrow_phase", "broad_phase", "ccd", "line_search"):
        t, c = avg(k)
        if t:
            out[k] = {"bound": "latency", "avg_launch_us": t * 1e6, "launches": c}
    return out


# ------------------------------------------------------------------------------ ours -------
def _stage_pass(P, s, steps):
    P.set_timing(s.h, True)
    P.kernel_times(s.h, reset=True)
    for _ in range(steps):
        s.step(n_iters=1)
    kt = P.kernel_times(s.h, reset=True)
    P.set_timing(s.h, False)
    return kt


def c3_single(P, local, steps):
    """Extra field: C3 single sequence (configs[2]) with its canonical actuation, frame F warm-
    started from the frame-(F-1) equilibrium computed like the batch's."""
    import torch
    import scenes
    sc = scenes.face_c3()
    s = P.Solver(sc, A=sc.actuation(TIMED_FRAME - 1)[None], device=local)
    s.step(n_iters=PREP_ITERS)
    s.step(A_next=sc.actuation(TIMED_FRAME)[None], n_iters=0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = None
    for _ in range(steps):
        st = s.step(n_iters=1)[0]
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    s.close()
    return {"workload": "C3: ~300k-tet two-slit face, canonical actuation 0.6 smoothstep, frame "
                        f"{TIMED_FRAME} warm-started (BASELINE.json configs[2])",
            "iters_per_s": steps / (ms / 1000.0), "ms_per_iter": ms / steps, "n_S_last": st["n_S"],
            "n_active_last": st["n_active"]}


def c2_extra(P, local, K):
    """Extra field: C2 (configs[1]) one sequence, frames 20.. warm-started, A on the device."""
    import numpy as np
    import torch
    import scenes
    sc = scenes.face_c2()
    frames = torch.from_numpy(np.stack([sc.actuation(f) for f in range(C2_FRAMES)])).to(f"cuda:{local}")
    s = P.Solver(sc, A=sc.actuation(0)[None], device=local, A_on_device=True)
    for f in range(C2_CONTACT_START):
        s.step(A_device_ptr=frames[f].data_ptr(), n_iters=ITERS_PER_FRAME)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(K):
        s.step(A_device_ptr=frames[min(C2_CONTACT_START + i, C2_FRAMES - 1)].data_ptr(), n_iters=ITERS_PER_FRAME)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    kt = _stage_pass(P, s, 20)
    s.close()
    return {"workload": "C2: face-like 47.5k-tet block, mouth slit (BASELINE.json configs[1])",
            "iters_per_s": K * ITERS_PER_FRAME / (ms / 1000.0),
            "frames_per_sec": K / (ms / 1000.0), "timed_frames": f"{C2_CONTACT_START}..{C2_CONTACT_START + K - 1}",
            "stage_us_per_launch": {k: round(v[0] / v[1] * 1000, 1) for k, v in kt.items() if v[1]}}


def _c5_local_step(size, hbm):
    import importlib.util
    spec = importlib.util.spec_from_file_location("c5_sweep", os.path.join(ROOT, "tools", "c5_sweep.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    r = mod.run(size)
    return {"workload": f"C5 pure-PD box {size} ({r['tets']} tets, {r['verts']} verts), 20-iteration steps "
                        "(BASELINE.json configs[4])",
            "local_step_GBps": r["local_step_GBps"], "local_step_frac": r["local_step_GBps"] / hbm,
            "gather_GBps": r["gather_GBps"], "gather_frac": r["gather_GBps"] / hbm,
            "pure_pd_iters_per_s": r["iters_per_s"], "peak_GBps": hbm,
            "bytes_per_tet": "local 240 (+32 per vertex), gather 28 per incidence + 40 per free vertex"}


def run_ours(a):
    import numpy as np
    import torch
    import torch.distributed as dist

    import scenes
    from paper_2312_02999_b200 import pd_ipc as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BENCH_SHARE_GPU=1 (correctness check of the multi-rank path on a 1-GPU box only: ranks share
    # device 0 and talk over gloo; its times are not a scaling measurement)
    share = os.environ.get("BENCH_SHARE_GPU") == "1"
    if share:
        local = local % torch.cuda.device_count()
    dev = f"cuda:{local}"
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    t_setup = time.perf_counter()
    sc = scenes.face_c3()
    mine = scenes.c4_assignment(a.seqs, rank, world)
    nb = len(mine)
    acts = [scenes.c4_actuation(sc, j) for j in mine]
    T, n = sc.n_tets, sc.n_verts
    A_prep = np.stack([f(TIMED_FRAME - 1) for f in acts])
    A_host = np.stack([f(TIMED_FRAME) for f in acts])
    K, W = a.steps, a.warmup
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)   # 256 MB > L2
    cpu_proc = None
    if world == 1 and not a.no_cpu_baseline:
        cpu_proc = start_cpu_baseline(mine[0], TIMED_FRAME - 1, a.cpu_seconds)

    # ---------------- device-resident run (value): the frame-F actuation is uploaded into the
    # handle BEFORE the timed region (pd_ipc_step with n_iters = 0), so the timed steps move no
    # host data
    s = P.Solver(sc, A=A_prep, n_seq=nb, device=local)
    info = P.get_info(s.h)
    s.step(n_iters=PREP_ITERS)                                          # untimed preparation
    for _ in range(W):                                                   # warm-up steps
        s.step(n_iters=1)
    s.step(A_next=A_host, n_iters=0)                                     # inputs resident in HBM
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    clocks = ClockSampler(local)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    stats = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    l0 = P.launch_count()
    t_wall = time.perf_counter()
    torch.cuda.nvtx.range_push("timed")                          # ncu --nvtx-include timed/
    for i in range(K):
        flush.fill_(float(i))                                    # evict L2 between steps
        ev[i][0].record()
        st = s.step(n_iters=1)
        ev[i][1].record()
        stats.append(st)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    launches = P.launch_count() - l0
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    my_ms = float(sum(e0.elapsed_time(e1) for e0, e1 in ev))
    checks = [(j, seq_checksum(s.positions(b))) for b, j in enumerate(mine)]
    nS_all = [st[b]["n_S"] for st in stats for b in range(nb)]
    nA_all = [st[b]["n_active"] for st in stats for b in range(nb)]
    reuse = sum(st[b]["sigma_reused"] for st in stats for b in range(nb)) / float(max(1, K * nb))
    upd = sum(st[b]["sigma_updated"] for st in stats for b in range(nb)) / float(max(1, K * nb))
    # exposed time of the reduced solve per sequence-iteration: B-check ready (end of the
    # sequence's assembly) -> dx ready (its Schur step + its share of the batched backward solves)
    exposed = statistics.mean(st[b]["ms"]["gstep"] for st in stats for b in range(nb))
    seq_ms = {k: statistics.mean(st[b]["ms"][k] for st in stats for b in range(nb))
              for k in ("ipc", "gstep", "ccd", "ls", "misc", "total")}

    # ---------------- end-to-end through the C ABI with host buffers (pinned): the same handle
    # continues frame F; every step copies the actuation of all the rank's sequences host ->
    # device (pd_ipc_step) and every sequence's positions device -> host (pd_ipc_positions)
    e2e = None
    if not a.no_e2e:
        pin = torch.empty(A_host.shape, dtype=torch.float64, pin_memory=True)
        pin.copy_(torch.from_numpy(A_host))
        pin_np = pin.numpy()
        xout = torch.empty((n, 3), dtype=torch.float64, pin_memory=True).numpy()
        Ke = min(K, E2E_STEPS)
        ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(Ke)]
        torch.cuda.synchronize()
        for i in range(Ke):
            flush.fill_(float(i))
            ev2[i][0].record()
            s.step(A_next=pin_np, n_iters=1)
            for b in range(nb):
                P.lib.pd_ipc_positions(s.h, b, xout.ctypes.data_as(P.C.POINTER(P.C.c_double)))
            ev2[i][1].record()
        torch.cuda.synchronize()
        e2e_ms = float(sum(e0.elapsed_time(e1) for e0, e1 in ev2))
        e2e = {"ms": e2e_ms, "h2d": nb * T * 9 * 8, "d2h": nb * n * 3 * 8, "steps": Ke}
    # per-kernel-group rooflines and the exposed reduced-solve time: a separate pass with every
    # group timed (timers in the timed region would cost time)
    kt = _stage_pass(P, s, 2)
    s.close()

    # ---------------- gather over ranks (NCCL): times, units, checksums
    cdev = "cpu" if share else dev
    allv = gather_rank_values([my_ms, e2e["ms"] if e2e else 0.0, float(nb * K),
                               float(nb * e2e["steps"]) if e2e else 0.0], world, cdev)
    by_seq = gather_checksums(checks, world, cdev, a.seqs)
    max_ms, max_e2e = float(allv[:, 0].max()), float(allv[:, 1].max())
    extras = {}
    if rank == 0 and world == 1 and not a.no_extras:
        extras["c3_single"] = c3_single(P, local, ITERS_PER_FRAME)
        extras["c2"] = c2_extra(P, local, 5)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    value = job_throughput(allv[:, 0], allv[:, 2])
    hbm, bf16, peak_src = _peaks()
    sm_max = _sm_max_mhz()
    rl_all = rooflines(kt, info, nb, nS_all, reuse, hbm, sm_max, peak_src, upd, nA_all)
    dom = rl_all.get("dense_schur")
    rl = None
    if dom:
        rl = {"bound": "tensor", "achieved": dom["achieved"], "peak": dom["peak"], "unit": "TFLOP/s",
              "frac": dom["frac"], "traffic": _traffic("k_schur_coop"), "kernel": "k_schur_coop",
              "flops_per_launch": dom["flops_per_launch"], "avg_launch_us": dom["avg_launch_us"],
              "peak_source": dom["peak_source"]}
    cpu = None
    if cpu_proc is not None:
        cpu = finish_cpu_baseline(cpu_proc, mine[0], TIMED_FRAME - 1)
    c5 = None
    if world == 1 and a.c5 and not a.no_extras:
        c5 = _c5_local_step(a.c5, hbm)
    units_total = float(allv[:, 2].sum())
    line = {
        "metric": "PD+IPC iterations/s", "value": value, "unit": "iters/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": max_ms / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators, SURVEY.md 8(d) C3 mesh + C4 actuations)",
        "frames_per_sec": value / ITERS_PER_FRAME,
        "config": {"workload": f"C4: {a.seqs} actuation sequences on the ~300k-tet two-slit face (C3 mesh), "
                               f"sharded j mod {world} (BASELINE.json configs[3])",
                   "tets": T, "verts": n, "surface_tris": int(sc.surf_tris.shape[0]),
                   "sequences_per_gpu": nb, "sequences_total": a.seqs,
                   "step": "one lockstep PD+IPC iteration of every sequence of the rank (20 steps = 1 frame)",
                   "timed": f"frame {TIMED_FRAME}, iterations 1..{K}, warm-started from the frame-"
                            f"{TIMED_FRAME - 1} state ({PREP_ITERS} untimed iterations from rest + {W} warm-up steps)",
                   "l2": "flushed between steps (256 MB write, outside the per-step CUDA events); the "
                         "batch's working set is also larger than L2",
                   "parallelism": f"dp{world} over independent sequences (no data-path collective)"},
        "roofline": rl,
        "rooflines": rl_all,
        "exposed_reduced_solve_ms_per_seq_iter": exposed,
        "stage_ms_per_seq_iter": seq_ms,
        "n_c_mean": statistics.mean(nS_all), "n_c_max": max(nS_all),
        "sigma_reuse_frac": reuse,
        "sigma_update_frac": upd,
        "cpu_baseline": cpu,
        "e2e": ({"value": float(allv[:, 3].sum()) / (max_e2e / 1000.0), "unit": "iters/s", "steps": e2e["steps"],
                 "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"],
                 "note": "every step: the actuation of all the rank's sequences copied from pinned host memory "
                         "(pd_ipc_step) and every sequence's positions copied back (pd_ipc_positions)"}
                if e2e else None),
        "gpu_launches": launches,
        "clocks": clk,
        "checksum": combined_checksum(by_seq),
        "checksum_note": "sha256 over the per-sequence position checksums in j order after the timed "
                         "steps: equal for every P iff every sequence's trajectory is bit-identical",
        "per_rank_ms": [float(v) for v in allv[:, 0]],
        "shared_gpu_check": share,
        "local_step_c5": c5,
        **extras,
        "info": info, "setup_s": t_setup, "wall_s": t_wall,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    a = _args()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
