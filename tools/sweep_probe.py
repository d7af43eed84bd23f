"""Time pdnn_weighted_levels (placement labels) on configs, with the debug
library's knobs (tools only; the product path never loads libpdnn_dbg.so).
    CFGS=2,3,4 VARIANTS='base;PDNN_SWEEP_NOWAIT=1;PDNN_SWEEP_CTAS=296' python tools/sweep_probe.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2008_08636_b200 import _binding, build
# VARIANT=name DEFS="A=1 B=2": a compile-time variant of the debug library
_defs = [d for d in os.environ.get("DEFS", "").split() if d]
_binding.load_library(build.build(debug_knobs=True, variant=os.environ.get("VARIANT", ""), defines=_defs))
from paper_2008_08636_b200 import Graph
from synth import make_config, candidate_parts

variants = [v for v in os.environ.get("VARIANTS", "base").split(";") if v]
for cfg in os.environ.get("CFGS", "2,3,4").split(","):
    w = make_config(int(cfg))
    G = Graph(w.V, w.src, w.dst); G.set_costs(w.c, w.w)
    part = torch.as_tensor(candidate_parts(w.seed, 0, 1, w.V, w.n_pe, "refine")[0].astype(np.int32)).cuda()
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    res = {"variant": os.environ.get("VARIANT", ""), "cfg": cfg, "V": w.V, "E": w.E, "D": G.n_levels}
    for var in variants:
        env = dict(kv.split("=") for kv in var.split(",") if "=" in kv)
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        for _ in range(3): G.weighted_levels(part)
        ts = []
        for _ in range(int(os.environ.get("REPS", "10"))):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); G.weighted_levels(part); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        for k, v in old.items():
            if v is None: os.environ.pop(k, None)
            else: os.environ[k] = v
        res[var] = round(float(np.median(ts)), 1)
    print(json.dumps(res), flush=True)
