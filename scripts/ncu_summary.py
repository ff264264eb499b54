"""Summarise an ncu report: key metrics + top stall lines + barrier-retry counts."""
import csv, subprocess, sys, io

rep = sys.argv[1]
def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))

rows = page("raw")
h, u, v = rows[0], rows[1], rows[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpc__cycles_elapsed.max"]
for k in keys:
    if k in h:
        i = h.index(k); print(f"{k:75s} {v[i]:>14s} {u[i]}")
rows = page("source", ["--print-source", "sass"])
h = rows[1]
si = h.index("Warp Stall Sampling (All Samples)"); ei = h.index("Instructions Executed")
stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
data = []
for r in rows[2:]:          # first kernel of the report only (a new header starts the next)
    if len(r) != len(h) or r[0] in ("Address", "Kernel Name"):
        break
    data.append(r)
tot = sum(float(r[si]) for r in data) or 1
print("--- top stall lines")
for r in sorted(data, key=lambda r: -float(r[si]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    reasons = sorted([(float(r[i]), h[i]) for i in stall_cols if r[i] not in ("", "0")], reverse=True)[:2]
    print(f"{float(r[si])/tot*100:5.1f}% {r[0][-5:]} {r[1].strip()[:58]:58s} x{r[ei]:>9s} {reasons}")
print("--- barrier waits / tensor instrs")
for r in data:
    if any(k in r[1] for k in ("TRYWAIT", "UTCHMMA", "LDTM")):
        print(f"{r[0][-5:]} {r[1].strip()[:70]:70s} exec={r[ei]}")
