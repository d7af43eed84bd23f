"""Device time of the C4 step: eager library calls vs one CUDA-graph replay per step (L2 flushed between steps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2008_08636_b200 import Graph
from synth import make_config, candidate_parts
w = make_config(4)
G = Graph(w.V, w.src, w.dst); G.set_costs(w.c, w.w)
part = torch.as_tensor(candidate_parts(w.seed, 0, 1, w.V, w.n_pe, "refine")[0].astype(np.int32)).cuda()
mem, kind, cap = (torch.as_tensor(x).cuda() for x in (w.mem, w.kind, w.cap_eff))
G.workspace()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def step():
    G.slice(1)
    tl, bl = G.weighted_levels(part)
    G.critical_path(tl, bl, part)
    G.memory_potential(part, w.n_pe, mem, kind, tl, cap)
for _ in range(3): step()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.graph(g, stream=s):
    step()
torch.cuda.current_stream().wait_stream(s)
def timeit(fn, n=20):
    ts = []
    for _ in range(n):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return np.median(ts), min(ts)
print("eager ms (median, min)", timeit(step))
print("graph ms (median, min)", timeit(g.replay))
