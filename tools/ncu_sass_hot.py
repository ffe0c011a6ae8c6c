"""Summarise an ncu source page (SASS): top instructions by executed count and stall samples."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
data = rows[2:]
tot_exec = sum(float(r[idx["Instructions Executed"]] or 0) for r in data)
tot_samp = sum(float(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print(f"total warp-instr {tot_exec:.3e}  stall samples {tot_samp:.0f}")
key = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
data.sort(key=lambda r: -float(r[idx[key]] or 0))
for r in data[:n]:
    print(f"{r[idx['Address']][-5:]} exec={float(r[idx['Instructions Executed']] or 0):.2e} samp={r[idx['Warp Stall Sampling (All Samples)']]:>6}  {r[idx['Source']].strip()[:90]}")
