"""Refinement timing probe (NEXT row N4, reading R22): pdnn_refine after
pdnn_slice_clusters + pdnn_lflam (CUDA events, after a warm-up call) beside the
oracle's or_refine on the same clusters and placement (configs up to
ORACLE_MAX_V nodes).  Usage: python tools/refine_probe.py [config ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import OracleGraph  # noqa: E402
from paper_2008_08636_b200 import Graph  # noqa: E402
from synth import make_config  # noqa: E402

ORACLE_MAX_V = int(os.environ.get("ORACLE_MAX_V", "70000"))
out = []
for n in [int(x) for x in sys.argv[1:]] or [6, 2, 3]:
    w = make_config(n)
    G = Graph(w.V, w.src, w.dst)
    G.set_costs(w.c, w.w)
    cof, mem, off, nc = G.slice_clusters(w.K)
    nc = int(nc.item())
    p0, _ = G.lflam(cof, mem, off, nc, w.K)
    G.refine(cof, mem, off, nc, w.K, p0)            # warm-up (workspace)
    torch.cuda.synchronize()
    ts = []
    for _ in range(2):
        t = time.perf_counter()
        part, log, L = G.refine(cof, mem, off, nc, w.K, p0)   # synchronous call
        ts.append(time.perf_counter() - t)
    og = OracleGraph(w.V, w.src, w.dst)
    p0h = p0.cpu().numpy()
    tl, bl = og.weighted_levels(w.c, w.w, p0h)
    r = {"config": w.name, "V": w.V, "D": int(og.levels().max()) + 1, "clusters": nc, "K": w.K,
         "swaps": int((log[:, 0] == 0).sum()) if len(log) else 0,
         "moves": int((log[:, 0] == 1).sum()) if len(log) else 0,
         "L_before": int((tl + bl).max()), "L_after": int(L), "gpu_s": round(min(ts), 4)}
    if w.V <= ORACLE_MAX_V:
        cof_h, mem_h, off_h = cof.cpu().numpy(), mem.cpu().numpy(), off.cpu().numpy()[: nc + 1]
        cl = [mem_h[off_h[i]:off_h[i + 1]] for i in range(nc)]
        t = time.perf_counter()
        part_o, log_o, L_o = og.refine(w.c, w.w, cof_h, cl, w.K, p0h)
        r["oracle_s"] = round(time.perf_counter() - t, 3)
        r["identical"] = bool(np.array_equal(part.cpu().numpy(), part_o) and log.tolist() == log_o.tolist()
                              and L == L_o)
    print(json.dumps(r), flush=True)
    out.append(r)
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/refine_probe.json", "w") as f:
    json.dump(out, f, indent=1)
