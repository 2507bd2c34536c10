#!/usr/bin/env python
"""Benchmark of the PD+IPC iteration (arXiv 2312.02999) on B200: prints ONE JSON line.

Workload (BASELINE.json configs[1]): synthetic face-like block of 47.5k tets
with a mouth slit, lips closing under actuation, 60 frames x 20 PD+IPC iterations.  A bench
"step" is one frame = 20 iterations of the whole hot path (local step, gather, broad/narrow
phase, contact assembly, contact-reduced global solve, CCD, line search, update).  The timed
frames are taken from the contact regime of the sequence (frames before it run untimed as
setup / warm-up, because frames are sequential: each starts from the previous equilibrium).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU (torchrun): one process per GPU, each rank simulates its own actuation sequence
(independent problems, no data-path collective: weak scaling); NCCL only carries the
per-rank timing / statistics; value = total iterations of all ranks / max-over-ranks time.
"""
from __future__ import annotations

import argparse
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
TIMED_GROUPS = ["local_step", "dense_schur"]      # the two roofline kernels (timers cost time)
N_FRAMES = 60
CONTACT_START = 20          # first frame of the timed window (lips in contact from ~frame 20)


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--c5", default="1M", help="pure-PD box size for the local-step HBM sweep ('' to skip)")
    return ap.parse_args()


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def _c5_local_step(size, hbm):
    """Local-step and gather HBM GB/s on the pure-PD box of BASELINE.json configs[4] (the metric's
    'local-step HBM GB/s' at a size where the step is bandwidth-relevant; C2 is latency-bound)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("c5_sweep", os.path.join(ROOT, "tools", "c5_sweep.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    r = mod.run(size)
    return {"workload": f"C5 pure-PD box {size} ({r['tets']} tets, {r['verts']} verts), 20-iteration steps",
            "local_step_GBps": r["local_step_GBps"], "local_step_frac": r["local_step_GBps"] / hbm,
            "gather_GBps": r["gather_GBps"], "gather_frac": r["gather_GBps"] / hbm,
            "pure_pd_iters_per_s": r["iters_per_s"], "peak_GBps": hbm,
            "bytes_per_tet": "local 240 (+32 per vertex), gather 28 per incidence + 40 per free vertex"}


def _sm_max_mhz():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["sm_max_mhz"])
    except Exception:
        return 1965.0


def _frame_index(f):
    return min(f, N_FRAMES - 1)


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


# ------------------------------------------------------------------------------ oracle -----
_CPU_SCRIPT = r"""
import json, sys, time
import numpy as np
sys.path.insert(0, sys.argv[1])
import scenes
from oracle import OracleSolver
sc = scenes.face_c2()
x = np.load(sys.argv[2])
frame = int(sys.argv[3]); budget = float(sys.argv[4])
o = OracleSolver(sc)
A = sc.actuation(frame)
t0 = time.perf_counter(); n = 0
while True:
    it = o.iterate(x, A); x = it["x"]; n += 1
    if time.perf_counter() - t0 >= budget: break
dt = time.perf_counter() - t0
print(json.dumps({"iters": n, "seconds": dt, "n_active": it["n_pt"] + it["n_ee"], "n_S": int(it["S"].size)}))
"""


def cpu_baseline(x_state, frame, budget):
    """The oracle as it stands, single thread, on a bounded sample of the same workload."""
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1",
               NUMEXPR_NUM_THREADS="1", CUDA_VISIBLE_DEVICES="")
    with tempfile.TemporaryDirectory() as td:
        xp = os.path.join(td, "x.npy")
        import numpy as np
        np.save(xp, x_state)
        sp = os.path.join(td, "cpu.py")
        with open(sp, "w") as f:
            f.write(_CPU_SCRIPT)
        r = subprocess.run([sys.executable, sp, ROOT, xp, str(frame), str(budget)], env=env,
                           capture_output=True, text=True, timeout=600)
    if r.returncode != 0:
        return {"value": None, "unit": "iters/s", "cores": 1, "kind": "oracle",
                "sample": "failed: " + r.stderr.strip().splitlines()[-1][:200]}
    d = json.loads(r.stdout.strip().splitlines()[-1])
    return {"value": d["iters"] / d["seconds"], "unit": "iters/s", "cores": 1, "kind": "oracle",
            "sample": f"{d['iters']} oracle iterations of C2 frame {frame} from the GPU state at the "
                      f"start of the timed window ({d['seconds']:.1f} s, |C| {d['n_active']}, "
                      f"n_c {d['n_S']}); full sparse LU of H-hat per iteration, 1 thread"}


# ------------------------------------------------------------------------------ reference --
def run_reference(a):
    """--impl reference: the CPU oracle, timed as it stands, on this arm's config and metric."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    import scenes
    from oracle import OracleSolver
    sc = scenes.face_c2()
    o = OracleSolver(sc)
    frame = CONTACT_START + 10
    A = sc.actuation(frame)
    x = sc.rest.copy()
    for _ in range(a.warmup):
        x = o.iterate(x, A)["x"]
    t0 = time.perf_counter()
    for _ in range(a.steps):
        it = o.iterate(x, A)
        x = it["x"]
    dt = time.perf_counter() - t0
    v = a.steps / dt
    line = {"impl": "reference", "metric": "PD+IPC iterations/s", "value": v, "unit": "iters/s",
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1000 * dt / a.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "frames_per_sec": v / ITERS_PER_FRAME,
            "config": {"workload": "C2: face-like 47.5k-tet block, mouth-slit lip contact "
                                   "(BASELINE.json configs[1])",
                       "step": "one oracle PD+IPC iteration (bounded sample)",
                       "sample": f"frame-{frame} actuation applied from rest; {a.warmup} untimed + "
                                 f"{a.steps} timed iterations"},
            "cpu_baseline": {"value": v, "unit": "iters/s", "cores": 1, "kind": "oracle",
                             "sample": f"{a.steps} oracle iterations (|C| {it['n_pt'] + it['n_ee']}, "
                                       f"n_c {int(it['S'].size)})"},
            "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ ours -------
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


def job_throughput(per_rank_ms, world, steps, iters_per_step=ITERS_PER_FRAME):
    """Whole-job iterations/s: every rank ran `steps` frames of its own sequence (weak scaling);
    the job took the slowest rank's time."""
    return world * steps * iters_per_step / (max(per_rank_ms) / 1000.0)


def run_ours(a):
    import numpy as np
    import torch
    import torch.distributed as dist

    import scenes
    from paper_2312_02999_b200 import pd_ipc as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sc = scenes.face_c2()
    T, n = sc.n_tets, sc.n_verts
    frames_host = np.stack([sc.actuation(f) for f in range(N_FRAMES)])      # (60, T, 9)
    frames_dev = torch.from_numpy(frames_host).to(f"cuda:{local}")
    K, W = a.steps, a.warmup
    start = max(CONTACT_START, W)
    timed = [start + i for i in range(K)]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")   # 256 MB

    # ---------------- device-resident run (value)
    s = P.Solver(sc, A=frames_host[0][None], device=local, A_on_device=True)
    for f in range(start - W):                                   # untimed setup frames
        s.step(A_device_ptr=frames_dev[_frame_index(f)].data_ptr(), n_iters=ITERS_PER_FRAME)
    for f in range(start - W, start):                            # warm-up frames
        s.step(A_device_ptr=frames_dev[_frame_index(f)].data_ptr(), n_iters=ITERS_PER_FRAME)
    x_start = s.positions()
    # live CUDA-event timers in the timed region only around the kernel groups the roofline needs
    # (an event pair per group per iteration is a graph node: timing every group costs ~15%)
    P.set_timing(s.h, True, groups=TIMED_GROUPS)
    P.kernel_times(s.h, reset=True)
    clocks = ClockSampler(local)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in timed]
    stats_log = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    l0 = P.launch_count()
    t_wall = time.perf_counter()
    torch.cuda.nvtx.range_push("timed")                          # ncu --nvtx-include timed/
    for i, f in enumerate(timed):
        flush.fill_(float(i))                                    # evict L2 between steps
        ev[i][0].record()
        st = s.step(A_device_ptr=frames_dev[_frame_index(f)].data_ptr(), n_iters=ITERS_PER_FRAME)
        ev[i][1].record()
        stats_log.append(st[0])
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    launches = P.launch_count() - l0
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    my_ms = float(sum(step_ms))
    ktimes = P.kernel_times(s.h, reset=True)
    # stage breakdown: every group timed, in a separate 2-frame pass after the timed region
    P.set_timing(s.h, True)
    for f in range(timed[-1] + 1, timed[-1] + 3):
        s.step(A_device_ptr=frames_dev[_frame_index(f)].data_ptr(), n_iters=ITERS_PER_FRAME)
    stages = P.kernel_times(s.h, reset=True)
    s.close()

    # ---------------- end-to-end through the C ABI with host buffers
    e2e = None
    if not a.no_e2e:
        pin = torch.empty((N_FRAMES, T, 9), dtype=torch.float64, pin_memory=True)
        pin.copy_(torch.from_numpy(frames_host))
        pin_np = pin.numpy()
        xout = torch.empty((n, 3), dtype=torch.float64, pin_memory=True).numpy()
        s2 = P.Solver(sc, A=frames_host[0][None], device=local)
        for f in range(start):
            s2.step(A_next=pin_np[_frame_index(f)][None], n_iters=ITERS_PER_FRAME)
        ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in timed]
        torch.cuda.synchronize()
        for i, f in enumerate(timed):
            flush.fill_(float(i))
            ev2[i][0].record()
            s2.step(A_next=pin_np[_frame_index(f)][None], n_iters=ITERS_PER_FRAME)
            P.lib.pd_ipc_positions(s2.h, 0, xout.ctypes.data_as(P.C.POINTER(P.C.c_double)))
            ev2[i][1].record()
        torch.cuda.synchronize()
        e2e_ms = float(sum(e0.elapsed_time(e1) for e0, e1 in ev2))
        s2.close()
        e2e = {"ms": e2e_ms, "h2d": T * 9 * 8, "d2h": n * 3 * 8}

    # ---------------- gather over ranks
    allv = gather_rank_values([my_ms, e2e["ms"] if e2e else 0.0], world, f"cuda:{local}")
    max_ms, max_e2e = float(allv[:, 0].max()), float(allv[:, 1].max())
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    iters_total = world * K * ITERS_PER_FRAME
    value = job_throughput(allv[:, 0], world, K)
    hbm, bf16, peak_src = _peaks()
    sm_max = _sm_max_mhz()
    # ---- roofline: dominant kernel group (live CUDA-event timings) and the local step
    name_dom = max(TIMED_GROUPS, key=lambda k: ktimes.get(k, (0.0, 0))[0])
    n_iter_timed = K * ITERS_PER_FRAME
    nS_mean = statistics.mean(st["n_S"] for st in stats_log)
    rl = _roofline(name_dom, ktimes, sc, hbm, sm_max, peak_src, stats_log)
    rl_local = _roofline("local_step", ktimes, sc, hbm, sm_max, peak_src, stats_log)
    cpu = None
    if world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(x_start, start, a.cpu_seconds)
    c5 = None
    if world == 1 and a.c5:
        c5 = _c5_local_step(a.c5, hbm)
    line = {
        "metric": "PD+IPC iterations/s", "value": value, "unit": "iters/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": max_ms / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, SURVEY.md 8(d) C2)",
        "frames_per_sec": world * K / (max_ms / 1000.0),
        "config": {"workload": "C2: face-like 47.5k-tet block, mouth-slit lip contact, 60 frames x "
                               "20 iterations (BASELINE.json configs[1])",
                   "tets": T, "verts": n, "surface_tris": int(sc.surf_tris.shape[0]),
                   "step": "one frame = 20 PD+IPC iterations",
                   "timed_frames": f"{timed[0]}..{timed[-1]} (contact regime; frames 0..{start - W - 1} "
                                   f"untimed setup, {start - W}..{start - 1} warm-up)",
                   "sequences_per_gpu": 1, "l2": "flushed between steps (256 MB write, outside the "
                                                 "per-step CUDA events)",
                   "parallelism": f"dp{world} over independent sequences"},
        "roofline": rl, "roofline_local_step": rl_local,
        "local_step_c5": c5,
        "cpu_baseline": cpu,
        "e2e": ({"value": iters_total / (max_e2e / 1000.0), "unit": "iters/s",
                 "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"]} if e2e else None),
        "gpu_launches": launches,
        "clocks": clk,
        "stage_ms_per_iter": {k: v[0] / max(v[1], 1) for k, v in stages.items() if v[1]},
        "stage_note": "stage_ms_per_iter from a separate 2-frame pass with every group timed; the timed "
                      "region times only " + ", ".join(TIMED_GROUPS),
        "n_c_mean": nS_mean, "n_active_last": stats_log[-1]["n_active"],
        "sigma_reuse_frac": sum(st["sigma_reused"] for st in stats_log) / float(K * ITERS_PER_FRAME),
        "alpha_last": stats_log[-1]["alpha"], "wall_s": t_wall,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# FP64 tensor (DMMA, mma.sync.m8n8k4.f64) throughput measured on this pool's B200 by
# tools/micro/fp64_peaks.cu: 128 flop/clk/SM (profiles/fp64_peaks_r01.txt).  tcgen05 has no
# f64 kind, so this is the FP64 contraction peak; x 148 SMs x the max SM clock.
DMMA_FLOP_PER_CLK_SM = 128.0
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


def _roofline(name, ktimes, sc, hbm, sm_max_mhz, peak_src, stats_log):
    """Achieved = algorithmic bytes (flops) per launch / average launch duration."""
    ms, cnt = ktimes.get(name, (0.0, 0))
    if cnt == 0 or ms <= 0:
        return None
    avg_s = ms / cnt / 1000.0
    T, n = sc.n_tets, sc.n_verts
    nf = n - len(sc.fixed)
    if name == "local_step":
        # per tet: tet ids 16 B, B_i 72, A_i (6 sym) 48, w_i 8, corner forces written 96;
        # per vertex: x 32 (double4) read once
        byts = T * (16 + 72 + 48 + 8 + 96) + n * 32
        return {"kernel": "k_local_step", "bound": "hbm", "achieved": byts / avg_s / 1e9, "peak": hbm,
                "unit": "GB/s", "frac": byts / avg_s / 1e9 / hbm, "traffic": _traffic("k_local_step"),
                "bytes_per_launch": byts, "avg_launch_us": avg_s * 1e6, "peak_source": peak_src}
    if name == "gather":
        byts = nf * (8 + 32) + 4 * T * (4 + 24)
        return {"kernel": "k_gather_elastic", "bound": "hbm", "achieved": byts / avg_s / 1e9, "peak": hbm,
                "unit": "GB/s", "frac": byts / avg_s / 1e9 / hbm, "traffic": _traffic("k_gather_elastic"),
                "bytes_per_launch": byts, "avg_launch_us": avg_s * 1e6, "peak_source": peak_src}
    if name == "dense_schur":
        # algorithmic flops of a9 at n_c = |S|, m = 3 n_c: Sigma_s = K^-1 (n_c^3), Cholesky of
        # the augmented Sigma-hat (m^3 / 3), back substitution 2 m^2, t = B u and Z 2 m^2
        nc = statistics.mean(st["n_S"] for st in stats_log)
        m = 3 * nc
        flops = nc ** 3 + m ** 3 / 3.0 + 4 * m ** 2
        fp64 = DMMA_FLOP_PER_CLK_SM * N_SM * sm_max_mhz * 1e6 / 1e12
        return {"kernel": "k_schur_coop", "bound": "tensor", "achieved": flops / avg_s / 1e12, "peak": fp64,
                "unit": "TFLOP/s", "frac": flops / avg_s / 1e12 / fp64, "traffic": _traffic("k_schur_coop"),
                "flops_per_launch": flops, "avg_launch_us": avg_s * 1e6,
                "peak_source": "FP64 DMMA measured (tools/micro/fp64_peaks.cu) x 148 SMs x max clock"}
    return {"kernel": name, "bound": "latency", "achieved": None, "peak": None, "unit": None,
            "frac": None, "traffic": None, "avg_launch_us": avg_s * 1e6,
            "note": "latency-bound stage; see DESIGN.md"}


def main():
    a = _args()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
