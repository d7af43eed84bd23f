"""Time the single-graph step's parts (slice(K), weighted_levels, critical_path,
memory_potential) per config with the debug library (knobs read from the
environment, e.g. PDNN_MERGE_MODE at graph build).  CFGS=3,8 python tools/step_probe.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2008_08636_b200 import _binding, build
_binding.load_library(build.build(debug_knobs=True))
from paper_2008_08636_b200 import Graph
from synth import make_config, candidate_parts
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cfg in os.environ.get("CFGS", "3,8").split(","):
    w = make_config(int(cfg))
    G = Graph(w.V, w.src, w.dst); G.set_costs(w.c, w.w)
    ps = torch.as_tensor(candidate_parts(w.seed, 0, 1, w.V, w.n_pe, "refine")[0].astype(np.int32)).cuda()
    m, k, c = (torch.as_tensor(x).cuda() for x in (w.mem, w.kind, w.cap_eff))
    K = max(w.K, 1)
    seg = []
    for rep in range(6):
        flush.zero_()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(); G.slice(K); ev[1].record()
        tl, bl = G.weighted_levels(ps); ev[2].record()
        G.critical_path(tl, bl, ps); ev[3].record()
        G.memory_potential(ps, w.n_pe, m, k, tl, c); ev[4].record()
        torch.cuda.synchronize()
        if rep >= 2: seg.append([ev[j].elapsed_time(ev[j + 1]) for j in range(4)])
    seg = np.array(seg)
    print(json.dumps({"cfg": cfg, "merge": os.environ.get("PDNN_MERGE_MODE"), "K": K,
                      "slice": [round(x, 3) for x in seg[:, 0]], "wl": [round(x, 3) for x in seg[:, 1]],
                      "cp": round(float(seg[:, 2].mean()), 3), "mem": round(float(seg[:, 3].mean()), 3)}), flush=True)
