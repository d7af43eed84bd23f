"""Warp-stall samples aggregated per CUDA source line (needs -lineinfo and
--import-source on).    python tools/ncu_lines.py REPORT KERNEL_REGEX [N]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kern,
                      "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
agg, src, cur = {}, {}, None
for r in rows:
    if len(r) <= i_s or r[0] == "Line No":
        continue
    if r[0]:
        cur = int(r[0]); src[cur] = r[1].strip()
        continue
    try:
        agg[cur] = agg.get(cur, 0) + int(r[i_s] or 0)
    except ValueError:
        pass
tot = sum(agg.values()) or 1
for ln, v in sorted(agg.items(), key=lambda x: -x[1])[:n]:
    print(f"{v / tot * 100:5.1f}%  L{ln:4d}  {src.get(ln, '')[:100]}")
