"""Per CUDA-source-line summary of an ncu report (needs -lineinfo and
--import-source on): instructions executed and warp-stall samples per line.

    python tools/ncu_lines.py report.ncu-rep [top_n] [sort: samp|exec]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
key = sys.argv[3] if len(sys.argv) > 3 else "samp"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = "?"
lines = []
tot_e = tot_s = 0.0
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No") or len(r) < 8:
        continue
    if r[0] != "" and r[2] == "-":
        s = float(r[4]) if r[4] not in ("-", "") else 0.0
        e = float(r[7]) if r[7] not in ("-", "") else 0.0
        tot_e += e
        tot_s += s
        if e or s:
            lines.append((fname, int(r[0]), r[1].strip(), e, s))
print(f"total warp-instr {tot_e:.3e}  stall samples {tot_s:.0f}")
lines.sort(key=lambda t: -(t[4] if key == "samp" else t[3]))
for f, ln, src, e, s in lines[:top]:
    print(f"{f}:{ln:<5d} exec={e:9.3e} ({100 * e / max(tot_e, 1):4.1f}%) samp={s:6.0f} ({100 * s / max(tot_s, 1):4.1f}%)  {src[:80]}")
