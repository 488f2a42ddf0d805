"""Summarise an ncu report: top SASS lines by stall samples, grouped by CUDA source line (tools only)."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
data = []
for r in rows:
    if "Warp Stall Sampling (All Samples)" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(r)
si = hdr.index("Warp Stall Sampling (All Samples)")
src_i = hdr.index("Source")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[si]) for r in data if r[si].isdigit())
print("total samples", tot)
for r in sorted(data, key=lambda r: -int(r[si]) if r[si].isdigit() else 0)[:n]:
    st = sorted([(int(r[i]), hdr[i][6:]) for i in stall_cols if r[i].isdigit() and int(r[i]) > 0], reverse=True)[:3]
    print(f"{int(r[si]):7d} {100*int(r[si])/tot:5.1f}%  {r[src_i][:70]:70s} {st}")
