"""Every library kernel on config 1 (and a hub graph for the batched hub
parts), for compute-sanitizer:  compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2008_08636_b200 import Graph
from synth import make_config, candidate_parts

w = make_config(1)
G = Graph(w.V, w.src, w.dst); G.set_costs(w.c, w.w)
part = candidate_parts(w.seed, 0, 1, w.V, w.n_pe)[0].astype(np.int32)
tl, bl = G.weighted_levels(part)
G.weighted_levels(None)
G.critical_path(tl, bl, part)
G.slice(2)
G.memory_potential(part, w.n_pe, w.mem, w.kind, tl, w.cap_eff, want_mcons=True)
parts = candidate_parts(w.seed, 0, 70, w.V, w.n_pe)
G.eval_batch(parts, w.n_pe, w.mem, w.kind, w.cap_eff)
G.eval_batch(parts[:40], w.n_pe, w.mem, w.kind, w.cap_eff, schedule=1)
G.emulate(part, w.n_pe)
G.validate(part=part, n_pe=w.n_pe, mem=w.mem, kind=w.kind, st=tl)
# NEXT rows: whole of Alg. 1, criticality, LFLAM, refinement, overflow handler
cof, mem_, off, nc = G.slice_clusters(w.K)
nc = int(nc.item())
G.criticality(cof, nc)
p0, _ = G.lflam(cof, mem_, off, nc, w.K)
G.refine(cof, mem_, off, nc, w.K, p0)
G.resolve_overflow(part, w.n_pe, w.mem, w.kind, np.asarray(w.cap_eff) // 2, max_moves=20)
# hubs (split parts in both sweeps)
n = 3000
src = np.concatenate([np.zeros(n - 2, np.int32), np.arange(1, n - 1, dtype=np.int32)])
dst = np.concatenate([np.arange(1, n - 1, dtype=np.int32), np.full(n - 2, n - 1, np.int32)])
H = Graph(n, src, dst); H.set_costs(np.arange(n, dtype=np.int64), np.ones(src.size, np.int64))
tl, bl = H.weighted_levels(np.zeros(n, np.int32))
H.critical_path(tl, bl, np.zeros(n, np.int32))
H.eval_batch(np.random.default_rng(0).integers(0, 4, (40, n)).astype(np.uint8), 4, np.ones(n, np.int64),
             np.zeros(n, np.uint8), np.full(4, 1 << 40, np.int64))
torch.cuda.synchronize()
print("sanitize run ok")
