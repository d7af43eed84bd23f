"""Executed warp instructions and stall samples per CUDA source line of one kernel.
    python tools/ncu_inst.py REPORT KERNEL_REGEX [N] [launch-skip]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kern,
                      "-s", skip, "-c", "1"], capture_output=True, text=True).stdout
data, hdr, fname = [], None, ""
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0].isdigit() and len(r) > 8:
        ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        try:
            data.append((f"{fname}:{r[0]}", r[1].strip(), float(r[ie] if r[ie] not in ("", "-") else 0),
                         float(r[st] if r[st] not in ("", "-") else 0)))
        except ValueError:
            pass
ti = sum(d[2] for d in data) or 1; ts = sum(d[3] for d in data) or 1
print(f"total inst {ti:.0f}")
for ln, src, i, s in sorted(data, key=lambda d: -d[2])[:n]:
    print(f"{ln:18s} inst {i / ti * 100:5.1f}%  stall {s / ts * 100:5.1f}%  {src[:80]}")
