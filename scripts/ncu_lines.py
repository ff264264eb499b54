"""Per CUDA-source-line stall samples of an ncu report (--print-source cuda,sass):
usage: python scripts/ncu_lines.py report.ncu-rep [top_n] [file_substring]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
want = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, rows = "", None, []
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        fname = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        rows.append((fname, r))
si = hdr.index("Warp Stall Sampling (All Samples)")
ei = hdr.index("Instructions Executed")
tot = sum(float(r[si] or 0) for _, r in rows) or 1.0
print(f"total samples {tot:.0f}")
for f, r in sorted(rows, key=lambda x: -float(x[1][si] or 0))[:top]:
    if want and want not in f:
        continue
    print(f"{float(r[si])/tot*100:5.1f}% {f.split('/')[-1]}:{r[0]:>5s} x{r[ei]:>9s}  {r[1].strip()[:90]}")
