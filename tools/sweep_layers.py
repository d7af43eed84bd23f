"""Single-graph sweep time on synthetic layered DAGs (width x depth, k random
predecessors in the previous level): separates hop latency from fan-in effects."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2008_08636_b200 import Graph
rng = np.random.default_rng(0)
for spec in os.environ.get("SPECS", "20000x64x1,20000x64x4,60x4000x1,60x4000x3").split(","):
    width, depth, k = (int(x) for x in spec.split("x"))
    V = width * depth
    src = []
    dst = []
    for l in range(1, depth):
        base, pb = l * width, (l - 1) * width
        for kk in range(k):
            if kk == 0:
                s_ = pb + np.arange(width)            # aligned predecessor (parallel chains)
            else:
                s_ = pb + rng.integers(0, width, width)
            src.append(s_); dst.append(base + np.arange(width))
    src = np.concatenate(src).astype(np.int64); dst = np.concatenate(dst).astype(np.int64)
    key = np.unique(src * V + dst)
    src = (key // V).astype(np.int32); dst = (key % V).astype(np.int32)
    G = Graph(V, src, dst); G.set_costs(rng.integers(0, 1000, V), rng.integers(0, 1000, src.size))
    part = torch.randint(0, 8, (V,), dtype=torch.int32, device=G.device)
    for _ in range(3): G.weighted_levels(part)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); G.weighted_levels(part); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    print(json.dumps({"spec": spec, "V": V, "E": int(src.size), "ms": ms, "us_per_level": ms * 1e3 / depth,
                      "GBps_alg": (24 * src.size + 48 * V) / ms / 1e6}), flush=True)
