"""Warp-stall samples and executed instructions aggregated per CUDA source line
(needs -lineinfo and --import-source on), over every source file of the kernel.
    python tools/ncu_lines.py REPORT KERNEL_REGEX [N] [launch index]"""
import csv, io, os, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kern,
                      "-s", skip, "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, inst, src = {}, {}, {}
fname, hdr = "?", None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1]); hdr = None
        continue
    if r[0] == "Line No":
        hdr = r
        i_s = hdr.index("Warp Stall Sampling (All Samples)")
        i_i = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) <= i_s or not r[0]:
        continue
    key = (fname, r[0])
    src[key] = r[1].strip()
    try:
        agg[key] = agg.get(key, 0) + int(r[i_s] or 0)
        inst[key] = inst.get(key, 0) + int(float(r[i_i] or 0))
    except ValueError:
        pass
tot = sum(agg.values()) or 1
itot = sum(inst.values()) or 1
print(f"total stall samples {tot}, warp instructions {itot}")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:n]:
    print(f"{v / tot * 100:5.1f}% stall {inst.get(k, 0) / itot * 100:5.1f}% inst  {k[0]}:{k[1]:>4}  {src.get(k, '')[:90]}")
print("-- by instructions")
for k, v in sorted(inst.items(), key=lambda x: -x[1])[:n]:
    print(f"{v / itot * 100:5.1f}% inst {agg.get(k, 0) / tot * 100:5.1f}% stall  {k[0]}:{k[1]:>4}  {src.get(k, '')[:90]}")
