"""Executed warp instructions and stall samples per CUDA source line of one kernel.
    python tools/ncu_inst.py REPORT KERNEL_REGEX [N] [launch-index]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda", "-k", "regex:" + kern,
                      "-s", skip, "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
ie = hdr.index("Instructions Executed"); st = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows:
    if len(r) > st and r[0].isdigit():
        try:
            data.append((int(r[0]), r[1].strip(), float(r[ie] or 0), float(r[st] or 0)))
        except ValueError:
            pass
ti = sum(d[2] for d in data) or 1; ts = sum(d[3] for d in data) or 1
print(f"total inst {ti:.0f}")
for ln, src, i, s in sorted(data, key=lambda d: -d[2])[:n]:
    print(f"L{ln:4d} inst {i / ti * 100:5.1f}%  stall {s / ts * 100:5.1f}%  {src[:90]}")
