import json, os, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2008_08636_b200 import _binding, build
_binding.load_library(build.build(debug_knobs=True))
from paper_2008_08636_b200 import Graph
from synth import make_config, candidate_parts
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
w = make_config(3)
G = Graph(w.V, w.src, w.dst); G.set_costs(w.c, w.w)
ps = torch.as_tensor(candidate_parts(w.seed, 0, 1, w.V, w.n_pe, "refine")[0].astype(np.int32)).cuda()
rng = np.random.default_rng(1)
un = np.full(w.V, -2, np.int32); un[rng.random(w.V) < 0.02] = -1
un = torch.as_tensor(un).cuda()
allun = torch.full((w.V,), -2, dtype=torch.int32, device="cuda")
res = {"merge": os.environ.get("PDNN_MERGE_MODE")}
for name, lab in [("none", None), ("place", ps), ("unassigned", allun), ("removed2pct", un)]:
    ts = []
    for rep in range(5):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); G.weighted_levels(lab); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res[name] = round(float(np.median(ts[1:])), 3)
t = []
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); G.slice(1); e1.record(); torch.cuda.synchronize(); t.append(e0.elapsed_time(e1))
res["slice1"] = round(min(t), 3)
t = []
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); G.slice(2); e1.record(); torch.cuda.synchronize(); t.append(e0.elapsed_time(e1))
res["slice2"] = round(min(t), 3)
print(json.dumps(res))
