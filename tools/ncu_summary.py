"""Per-kernel summary of an ncu report (`ncu -i REPORT --page raw --csv`): duration, DRAM bytes
and throughput, SM / FP64 / DMMA pipe utilisation, occupancy, registers, top stall reasons.
Usage: python tools/ncu_summary.py REPORT.ncu-rep [--traffic-json OUT.json]"""
import csv
import io
import json
import subprocess
import sys

COLS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_B": "dram__bytes_read.sum",
    "dram_write_B": "dram__bytes_write.sum",
    "dram_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "dmma_pipe_pct": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}
SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def rows(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def main():
    report = sys.argv[1]
    hdr, units, data = rows(report)
    idx = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("smsp__average_warp_latency_issue_stalled_")
                  and h.endswith(".ratio")] or \
                 [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
    traffic = {}
    for r in data:
        name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "").replace("pdipc::", "")
        vals = {}
        for k, col in COLS.items():
            if col not in idx:
                continue
            v = r[idx[col]].replace(",", "")
            try:
                x = float(v) * SCALE.get(units[idx[col]], 1.0)
            except ValueError:
                continue
            if k == "duration_us":
                x = float(v) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0,
                                "ms": 1e3, "msecond": 1e3}.get(units[idx[col]], 1e-3)
            vals[k] = x
        st = []
        for c in stall_cols:
            try:
                st.append((float(r[idx[c]].replace(",", "")), c.split("stalled_")[1].split(".")[0]))
            except ValueError:
                pass
        st.sort(reverse=True)
        print(f"== {name}")
        for k, v in vals.items():
            print(f"   {k:15s} {v:,.3f}")
        if st:
            tot = sum(x for x, _ in st) or 1.0
            print("   top stalls:   " + ", ".join(f"{n} {100 * x / tot:.0f}%" for x, n in st[:5]))
        if "dram_read_B" in vals and "dram_write_B" in vals:
            traffic.setdefault(name, vals["dram_read_B"] + vals["dram_write_B"])
    if "--traffic-json" in sys.argv:
        with open(sys.argv[sys.argv.index("--traffic-json") + 1], "w") as f:
            json.dump(traffic, f, indent=1)


if __name__ == "__main__":
    main()
