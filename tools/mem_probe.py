"""Time pdnn_memory_potential (single placement) on configs through the debug
library (compile-time variants: VARIANT / DEFS as tools/sweep_probe.py)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2008_08636_b200 import _binding, build
_binding.load_library(build.build(debug_knobs=True, variant=os.environ.get("VARIANT", ""),
                                  defines=[d for d in os.environ.get("DEFS", "").split() if d]))
from paper_2008_08636_b200 import Graph
from synth import make_config, candidate_parts
for cfg in os.environ.get("CFGS", "3,4").split(","):
    w = make_config(int(cfg))
    G = Graph(w.V, w.src, w.dst); G.set_costs(w.c, w.w)
    part = torch.as_tensor(candidate_parts(w.seed, 0, 1, w.V, w.n_pe, "refine")[0].astype(np.int32)).cuda()
    tl, bl = G.weighted_levels(part)
    mem, kind, cap = (torch.as_tensor(x).cuda() for x in (w.mem, w.kind, w.cap_eff))
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    for _ in range(3): G.memory_potential(part, w.n_pe, mem, kind, tl, cap)
    ts = []
    for _ in range(10):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); G.memory_potential(part, w.n_pe, mem, kind, tl, cap); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(json.dumps({"variant": os.environ.get("VARIANT", ""), "cfg": cfg, "us_med": round(float(np.median(ts)), 1)}), flush=True)
