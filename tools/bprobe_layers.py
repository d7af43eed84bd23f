"""Batched sweep (+ CP walk) on synthetic layered DAGs: SPECS = width x depth x
k (k predecessors per node in the previous level, the first one aligned),
B candidates; PDNN_BATCH_NO_MEM=1 times the candidate-parallel sweep + CP only."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2008_08636_b200 import Graph
rng = np.random.default_rng(0)
B = int(os.environ.get("B", "32"))
for spec in os.environ.get("SPECS", "1x4000x1,60x4000x1,60x4000x3").split(","):
    width, depth, k = (int(x) for x in spec.split("x"))
    V = width * depth
    src, dst = [], []
    for l in range(1, depth):
        base, pb = l * width, (l - 1) * width
        for kk in range(k):
            s_ = pb + (np.arange(width) if kk == 0 else rng.integers(0, width, width))
            src.append(s_); dst.append(base + np.arange(width))
    src = np.concatenate(src).astype(np.int64); dst = np.concatenate(dst).astype(np.int64)
    key = np.unique(src * V + dst)
    src = (key // V).astype(np.int32); dst = (key % V).astype(np.int32)
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
    print(json.dumps({"spec": spec, "B": B, "ms": min(ts), "us_per_level": min(ts) * 1e3 / depth}), flush=True)
