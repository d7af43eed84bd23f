"""Summarise an ncu launch list (gpu__time_duration.sum per launch) for the last bench step."""
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
starts = [i for i, (_, k, _) in enumerate(data) if "k_labels" in k]
last = data[starts[-2]:] if len(starts) >= 2 else data   # slice's label fill starts a step
tot = 0.0
for _, k, v in last:
    if k.startswith("void at::") or k.startswith("at::"):
        continue
    tot += v
    print(f"{v/1e3:9.1f} us  {k[:90]}")
print(f"total {tot/1e3:.1f} us over {len(last)} launches")
