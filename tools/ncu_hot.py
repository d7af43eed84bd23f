"""Top stalled SASS instructions (and their CUDA source lines) of one kernel in an ncu report.
    python tools/ncu_hot.py REPORT KERNEL_REGEX [N]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
def page(kind):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern, "-c", "1",
                          "--print-source", kind], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))
rows = page("sass")
hdr = rows[1]; data = rows[2:]
i_src = hdr.index("Source"); i_s = hdr.index("Warp Stall Sampling (All Samples)")
data = [r for r in data if len(r) > i_s and (r[i_s] or "0").isdigit()]
tot = sum(int(r[i_s] or 0) for r in data)
print("total samples", tot, "instructions", len(data))
for idx, r in sorted(enumerate(data), key=lambda x: -int(x[1][i_s] or 0))[:n]:
    print(f"{idx:5d} {int(r[i_s]) / tot * 100:5.1f}%  {r[i_src].strip()[:100]}")
