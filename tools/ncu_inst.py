"""Instructions executed per CUDA source line from an ncu report (tools only)."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Instructions Executed" in r)
ii, si, li = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Line No") if "Line No" in hdr else 0
data = [r for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr) and r[ii].replace('.', '').isdigit()]
tot = sum(float(r[ii]) for r in data)
print(f"total warp-instructions {tot:.3e}")
for r in sorted(data, key=lambda r: -float(r[ii]))[:n]:
    print(f"{float(r[ii]):11.0f} {100*float(r[ii])/tot:5.1f}%  L{r[li]:>4s} {r[si].strip()[:90]}")
