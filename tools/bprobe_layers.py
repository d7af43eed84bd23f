"""Hop latency of the batched sweep on synthetic layered DAGs (width x depth),
each node reading 1-3 random nodes of the previous level; PDNN_BATCH_NO_MEM=1
recommended.  Reports ms per sweep+CP launch and us per level."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2008_08636_b200 import Graph
rng = np.random.default_rng(0)
B = int(os.environ.get("B", "32"))
for width in [int(x) for x in os.environ.get("WIDTHS", "1,8,64").split(",")]:
    depth = int(os.environ.get("DEPTH", "4000"))
    V = width * depth
    src, dst = [], []
    for l in range(1, depth):
        for j in range(width):
            v = l * width + j
            k = min(width, int(rng.integers(1, 4)))
            for u in rng.choice(width, k, replace=False):
                src.append((l - 1) * width + int(u)); dst.append(v)
    src = np.array(src, np.int32); dst = np.array(dst, np.int32)
    G = Graph(V, src, dst); G.set_costs(rng.integers(0, 1000, V), rng.integers(0, 1000, src.size))
    mem = torch.ones(V, dtype=torch.int64, device=G.device); kind = torch.zeros(V, dtype=torch.uint8, device=G.device)
    cap = torch.full((4,), 1 << 40, dtype=torch.int64, device=G.device)
    parts = torch.randint(0, 4, (B, V), dtype=torch.uint8, device=G.device)
    out = G.eval_batch(parts, 4, mem, kind, cap)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); G.eval_batch(parts, 4, mem, kind, cap, out=out); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(json.dumps({"width": width, "depth": depth, "B": B, "ms": min(ts), "us_per_level": min(ts) * 1e3 / depth}), flush=True)
