"""Repeat the single-placement memory tracker and a batched evaluation many times and
check every repetition is bit-identical to the first (races in the look-back scan,
the chunked sort's barriers or the segmented sort's prefetch would show up here)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2008_08636_b200 import Graph
from synth import make_config, candidate_parts
reps = int(os.environ.get("REPS", "40"))
for cfg in (4, 2):
    w = make_config(cfg)
    G = Graph(w.V, w.src, w.dst); G.set_costs(w.c, w.w)
    part = torch.as_tensor(candidate_parts(w.seed, 0, 1, w.V, w.n_pe, "refine")[0].astype(np.int32)).cuda()
    tl, _ = G.weighted_levels(part)
    ref = {k: v.clone() for k, v in G.memory_potential(part, w.n_pe, w.mem, w.kind, tl, w.cap_eff).items() if v is not None}
    for r in range(reps):
        got = G.memory_potential(part, w.n_pe, w.mem, w.kind, tl, w.cap_eff)
        for k, v in ref.items():
            assert torch.equal(got[k], v), (cfg, r, k)
    print("memory", cfg, "ok", reps)
w = make_config(5)
G = Graph(w.V, w.src, w.dst); G.set_costs(w.c, w.w)
parts = torch.as_tensor(candidate_parts(w.seed, 0, 256, w.V, w.n_pe, "uniform")).cuda()
ref = G.eval_batch(parts, w.n_pe, w.mem, w.kind, w.cap_eff).clone()
for r in range(max(reps // 4, 3)):
    got = G.eval_batch(parts, w.n_pe, w.mem, w.kind, w.cap_eff)
    assert torch.equal(got, ref), ("batch", r)
print("batch ok")
