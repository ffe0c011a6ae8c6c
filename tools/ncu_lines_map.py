"""Aggregate an ncu source page's stall samples / executed instructions per CUDA
source line, using nvdisasm line info of the same binary.
    python tools/ncu_lines_map.py REPORT.ncu-rep BINARY KERNEL_MANGLED_SUBSTR [N]"""
import csv, os, re, subprocess, sys, tempfile
rep, binary, kname = sys.argv[1:4]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(binary)], cwd=d, capture_output=True)
sass = ""
for cub in sorted(f for f in os.listdir(d) if f.endswith(".cubin")):
    names = subprocess.run(["cuobjdump", "-symbols", os.path.join(d, cub)], capture_output=True, text=True).stdout
    if kname in names:
        sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
        break
cur, a2l, inside = None, {}, False
for ln in sass.splitlines():
    if ln.startswith(".text.") or ln.startswith("//---------------------"):
        if ".text." in ln:
            inside = kname in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        a2l[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0] if rows[0][0] == "Address" else rows[1]
ix = {k: i for i, k in enumerate(h)}
data = [r for r in rows if r and r[0] != "Address" and re.match(r"0x", r[0] or "")]
base = int(data[0][ix["Address"]], 16)
agg = {}
tot_s = tot_e = 0.0
for r in data:
    key = a2l.get(int(r[ix["Address"]], 16) - base, ("?", 0))
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    e = float(r[ix["Instructions Executed"]] or 0)
    a = agg.setdefault(key, [0.0, 0.0])
    a[0] += s; a[1] += e; tot_s += s; tot_e += e
print(f"{len(a2l)} SASS lines mapped; samples {tot_s:.0f}, warp-instr {tot_e:.0f}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
    print(f"{v[0]:7.0f} {v[1]:8.0f}  {k[0]}:{k[1]}")
