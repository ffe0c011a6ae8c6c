"""Summarise `ncu --set full` reports into one markdown table (duration,
DRAM bytes, achieved HBM GB/s and fraction of the measured peak, occupancy,
top warp-stall reasons) + the launch lists' per-kernel shares of a step.

    python tools/ncu_summary.py gpurun_out/r2ncu > profiles/r2/ncu/summary.md
"""
import csv
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STALLS = ["long_scoreboard", "barrier", "wait", "short_scoreboard", "no_instructions", "branch_resolving",
          "math_pipe_throttle", "mio_throttle", "lg_throttle", "selected", "not_selected", "membar", "sleeping"]


def peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6650.0


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return None
    h, units, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    return d, u


def num(d, k):
    try:
        return float(str(d.get(k, "nan")).replace(",", ""))
    except ValueError:
        return float("nan")


def to_bytes(val, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return val * scale.get(unit, 1)


def to_us(val, unit):
    scale = {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}
    return val * scale.get(unit, 1e-3)


def main():
    d0 = sys.argv[1]
    pk = peak()
    print(f"| capture | kernel | time (us) | DRAM read+write (MB) | HBM GB/s | of {pk:.0f} GB/s | warps active % | "
          f"top stalls (share of samples) |")
    print("|---|---|---|---|---|---|---|---|")
    for rep in sorted(glob.glob(os.path.join(d0, "*.ncu-rep"))):
        r = raw(rep)
        name = os.path.basename(rep)[:-8]
        if r is None:
            print(f"| {name} | (no kernel captured) | | | | | | |")
            continue
        d, u = r
        t = to_us(num(d, "gpu__time_duration.sum"), u.get("gpu__time_duration.sum", "nsecond"))
        rd = to_bytes(num(d, "dram__bytes_read.sum"), u.get("dram__bytes_read.sum", "byte"))
        wr = to_bytes(num(d, "dram__bytes_write.sum"), u.get("dram__bytes_write.sum", "byte"))
        gbs = (rd + wr) / (t * 1e-6) / 1e9 if t > 0 else float("nan")
        occ = num(d, "sm__warps_active.avg.pct_of_peak_sustained_active")
        st = {s: num(d, f"smsp__pcsamp_warps_issue_stalled_{s}") for s in STALLS}
        tot = sum(v for v in st.values() if v == v)
        top = sorted(((v, s) for s, v in st.items() if v == v and v > 0), reverse=True)[:3]
        tops = ", ".join(f"{s} {100 * v / tot:.0f}%" for v, s in top) if tot else ""
        kname = d.get("Kernel Name", d.get("kernel_name", "?"))
        kname = kname.split("(")[0].replace("void ", "")[:60]
        print(f"| {name} | `{kname}` | {t:.1f} | {(rd + wr) / 1e6:.1f} | {gbs:.0f} | {gbs / pk:.3f} | {occ:.1f} | {tops} |")
    for f in sorted(glob.glob(os.path.join(d0, "launches_*.csv"))):
        rows = list(csv.reader(open(f)))
        h = None
        per = {}
        for r in rows:
            if "Kernel Name" in r:
                h = {k: i for i, k in enumerate(r)}
                continue
            if h and len(r) > max(h.values()) and r[h["Metric Name"]] == "gpu__time_duration.sum":
                k = r[h["Kernel Name"]].split("(")[0].replace("void ", "")
                per.setdefault(k, []).append(num({"x": r[h["Metric Value"]]}, "x"))
        print(f"\n{os.path.basename(f)} (ncu, serialised, cold caches): per-kernel mean duration and share")
        tot = sum(sum(v) for v in per.values())
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            print(f"- `{k[:70]}`: {len(v)} launches, mean {sum(v) / len(v) / 1e3:.1f} us, {100 * sum(v) / tot:.1f}%")


if __name__ == "__main__":
    main()
