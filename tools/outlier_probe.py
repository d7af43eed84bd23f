"""Repeat the single-graph step on a config many times and report each rep's
placement-sweep / tracker time (hunting rare slow reps).  CFGS=7,8 REPS=30"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2008_08636_b200 import Graph
from synth import make_config, candidate_parts
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cfg in os.environ.get("CFGS", "7,8").split(","):
    w = make_config(int(cfg))
    G = Graph(w.V, w.src, w.dst); G.set_costs(w.c, w.w)
    ps = torch.as_tensor(candidate_parts(w.seed, 0, 1, w.V, w.n_pe, "refine")[0].astype(np.int32)).cuda()
    m, k, c = (torch.as_tensor(x).cuda() for x in (w.mem, w.kind, w.cap_eff))
    K = max(w.K, 1)
    wl, mm = [], []
    for rep in range(int(os.environ.get("REPS", "30"))):
        flush.zero_()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(); G.slice(K); ev[1].record()
        tl, bl = G.weighted_levels(ps); ev[2].record()
        G.critical_path(tl, bl, ps); ev[3].record()
        G.memory_potential(ps, w.n_pe, m, k, tl, c); ev[4].record()
        torch.cuda.synchronize()
        wl.append(round(ev[1].elapsed_time(ev[2]), 3)); mm.append(round(ev[3].elapsed_time(ev[4]), 3))
    print(json.dumps({"cfg": cfg, "wl": wl, "mem": mm}), flush=True)
    del G
    torch.cuda.empty_cache()
