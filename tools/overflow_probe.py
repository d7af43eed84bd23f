"""Overflow-handler timing probe (NEXT row N3): pdnn_resolve_overflow (a host
loop over the library's kernels) beside the oracle's or_resolve_overflow on
the same placement and capacities.  Usage: python tools/overflow_probe.py"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import OracleGraph
from paper_2008_08636_b200 import Graph
from synth import candidate_parts, make_config
out = []
for n, scale, mm in [(2, 1.0, 40), (3, 1.6, 40), (4, 1.0, 10)]:
    w = make_config(n)
    G = Graph(w.V, w.src, w.dst); G.set_costs(w.c, w.w)
    part0 = candidate_parts(w.seed, 0, 1, w.V, w.n_pe, "refine")[0].astype(np.int32)
    cap = (w.cap_eff * scale).astype(np.int64)
    G.resolve_overflow(part0, w.n_pe, w.mem, w.kind, cap, max_moves=2)   # warm-up
    torch.cuda.synchronize()
    t = time.perf_counter()
    part, moves, res = G.resolve_overflow(part0, w.n_pe, w.mem, w.kind, cap, max_moves=mm)
    tg = time.perf_counter() - t
    og = OracleGraph(w.V, w.src, w.dst)
    t = time.perf_counter()
    want_part, want_moves, want_res = og.resolve_overflow(w.c, w.w, w.mem, w.kind, w.n_pe, cap, part0, max_moves=mm)
    to = time.perf_counter() - t
    r = {"config": w.name, "V": w.V, "decisions": len(moves), "moved": int((moves[:, 2] >= 0).sum()) if len(moves) else 0,
         "resolved": bool(res), "gpu_s": round(tg, 4), "oracle_s": round(to, 3),
         "identical": bool(res == want_res and np.array_equal(moves, want_moves)
                           and np.array_equal(part.cpu().numpy(), want_part))}
    print(json.dumps(r), flush=True)
    out.append(r)
