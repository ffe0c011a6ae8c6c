"""Print SASS in address order with exec counts, collapsing cold stretches."""
import csv, subprocess, sys
rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 1e6
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; idx = {k: i for i, k in enumerate(h)}
data = rows[2:]
acc = 0.0; samp = 0
for r in data:
    e = float(r[idx["Instructions Executed"]] or 0); s = int(float(r[idx["Warp Stall Sampling (All Samples)"]] or 0))
    if e >= thr or s > 300:
        if acc: print(f"   ... {acc:.2e} instr, {samp} samples")
        acc = 0; samp = 0
        print(f"{r[idx['Address']][-5:]} {e:9.2e} {s:6d}  {r[idx['Source']].strip()[:100]}")
    else:
        acc += e; samp += s
print(f"   ... {acc:.2e} instr, {samp} samples")
