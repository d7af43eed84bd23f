"""Time pdnn_eval_batch on config 5 (TRN graph) for a few batch sizes; check a
sample of candidates against the oracle.  PDNN_BATCH_NO_MEM=1 times the
candidate-parallel sweep + CP only."""
import os, sys, json, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import make_config, candidate_parts
if os.environ.get("VARIANT") or os.environ.get("DEFS") or os.environ.get("PDNN_DBG"):   # debug library (knobs, variants)
    from paper_2008_08636_b200 import _binding, build
    _binding.load_library(build.build(debug_knobs=True, variant=os.environ.get("VARIANT", ""),
                                      defines=[d for d in os.environ.get("DEFS", "").split() if d]))
from paper_2008_08636_b200 import Graph
w = make_config(int(os.environ.get("CFG", "5")))
G = Graph(w.V, w.src, w.dst); G.set_costs(w.c, w.w)
dev = G.device
mem, kind, cap = (torch.as_tensor(x).to(dev) for x in (w.mem, w.kind, w.cap_eff))
for B in [int(x) for x in os.environ.get("BS", "32,256,1024,4096").split(",")]:
    parts = torch.as_tensor(candidate_parts(w.seed, 0, B, w.V, w.n_pe, "uniform")).to(dev)
    out = G.eval_batch(parts, w.n_pe, mem, kind, cap)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); G.eval_batch(parts, w.n_pe, mem, kind, cap, out=out); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(json.dumps({"B": B, "ms": min(ts), "evals_per_s": B / min(ts) * 1e3, "no_mem": bool(os.environ.get("PDNN_BATCH_NO_MEM")),
                      "D": G.n_levels}), flush=True)
