"""Stall breakdown + instruction counts for an address range of the SASS source page."""
import csv, subprocess, sys, io, collections
rep, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
si = h.index("Warp Stall Sampling (All Samples)"); ei = h.index("Instructions Executed")
stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
data = [r for r in rows[2:] if len(r) == len(h)]
sel = [r for r in data if lo <= int(r[0], 16) & 0xFFFFF < hi]
tot = collections.Counter()
ins = 0
for r in sel:
    ins += int(r[ei] or 0)
    for i in stall_cols:
        if r[i] not in ("", "0"):
            tot[h[i]] += float(r[i])
print("instructions executed in range:", ins, " samples:", sum(float(r[si]) for r in sel))
for k, v in tot.most_common(10):
    print(f"  {k:40s} {v:8.0f}")
