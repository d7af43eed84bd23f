"""Summarise an ncu launch list (gpu__time_duration.sum per launch) for the last
bench step: the step is the trailing repeat of the launch sequence (the
L2-flush fill kernels of bench.py are dropped first)."""
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
data = []
for r in rows[1:]:
    try:
        data.append((int(r[ii]), r[ki], float(r[vi].replace(",", ""))))
    except ValueError:
        pass
data = [d for d in data if not (d[1].startswith("void at::") or d[1].startswith("at::"))]
names = [k for _, k, _ in data]
# smallest period p such that the last p launches repeat the p before them
last = data
for p in range(1, len(names) // 2 + 1):
    if names[-p:] == names[-2 * p:-p]:
        last = data[-p:]
        break
tot = 0.0
for _, k, v in last:
    tot += v
    print(f"{v/1e3:9.1f} us  {k[:90]}")
print(f"total {tot/1e3:.1f} us over {len(last)} launches")
