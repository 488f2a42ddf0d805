"""Per-CUDA-source-line instruction counts and stall samples from an ncu report (tools only)."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
div = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r)
hdr = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[2] == "-"]  # CUDA-line rows
ii = hdr.index("Instructions Executed")
si = hdr.index("Warp Stall Sampling (All Samples)")
f = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
tot_i = sum(f(r[ii]) for r in data)
tot_s = sum(f(r[si]) for r in data)
print(f"total warp-instructions {tot_i:.3e} (per unit {tot_i/div:.0f}); samples {tot_s:.0f}")
for r in sorted(data, key=lambda r: -f(r[ii]))[:top]:
    print(f"{r[0]:>5} {f(r[ii])/div:9.1f} instr {100*f(r[si])/max(tot_s,1):5.1f}% stall  {r[1].strip()[:95]}")
