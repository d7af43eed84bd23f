"""Per-item timestamps of one placement sweep (debug library, PDNN_SWEEP_TRACE=1):
per level, when its last item published (hop = difference), and per item the
split start -> inputs ready -> published.    CFG=4 python tools/sweep_trace.py"""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2008_08636_b200 import _binding, build
lib = _binding.load_library(build.build(debug_knobs=True, variant=os.environ.get("VARIANT", ""),
                                        defines=[d for d in os.environ.get("DEFS", "").split() if d]))
from paper_2008_08636_b200 import Graph
from synth import make_config, candidate_parts
lib.pdnn_debug_sweep_items.argtypes = [C.c_void_p, C.c_void_p]
lib.pdnn_debug_sweep_trace.argtypes = [C.c_void_p, C.c_int64]
w = make_config(int(os.environ.get("CFG", "4")))
G = Graph(w.V, w.src, w.dst); G.set_costs(w.c, w.w)
part = torch.as_tensor(candidate_parts(w.seed, 0, 1, w.V, w.n_pe, "refine")[0].astype(np.int32)).cuda()
os.environ["PDNN_SWEEP_TRACE"] = "1"
for _ in range(3): G.weighted_levels(part)
torch.cuda.synchronize()
ni = lib.pdnn_debug_sweep_items(G.handle, None)
it = np.zeros((ni, 4), dtype=np.int32)
assert lib.pdnn_debug_sweep_items(G.handle, it.ctypes.data) == 0
tr = np.zeros((ni, 3), dtype=np.uint64)
assert lib.pdnn_debug_sweep_trace(tr.ctypes.data, 3 * ni) == 0
lvl_by_rank = np.sort(G.levels().cpu().numpy())
fwd = it[:, 0] >= 0
r0 = np.where(fwd, it[:, 0], ~it[:, 0])
lv = np.where((it[:, 3] & (1 << 30)) != 0, 0, lvl_by_rank[np.minimum(r0, len(lvl_by_rank) - 1)])   # indexed items: level 0
t0 = tr[:, 2][tr[:, 2] > 0].min()
t = (tr.astype(np.int64) - int(t0)) / 1e3   # us
thread = it[:, 1] > 0
out = {"cfg": os.environ.get("CFG", "4"), "items": int(ni), "D": int(lvl_by_rank.max() + 1),
       "total_us": float(t[:, 2].max())}
for d, name in ((True, "tl"), (False, "bl")):
    m = fwd == d
    levels = np.unique(lv[m])
    done = np.array([t[m & (lv == l), 2].max() for l in levels])
    order = levels if d else levels[::-1]
    dd = np.array([t[m & (lv == l), 2].max() for l in order])
    done_by_level = [round(float(x), 2) for x in dd]
    hops = np.diff(dd)
    sel = m & thread
    proc = t[sel, 2] - t[sel, 1]
    wait = t[sel, 1] - t[sel, 0]
    # how long after its previous level's completion an item publishes
    prev_done = {}
    for k in range(1, len(order)):
        prev_done[order[k]] = dd[k - 1]
    lag = np.array([t[i, 2] - prev_done[lv[i]] for i in np.nonzero(sel)[0] if lv[i] in prev_done])
    start_lag = np.array([t[i, 0] - prev_done[lv[i]] for i in np.nonzero(sel)[0] if lv[i] in prev_done])
    q = lambda a: [round(float(np.percentile(a, p)), 2) for p in (10, 50, 90, 99, 100)] if len(a) else []
    out[name] = {"hop_us": q(hops), "hop_sum": round(float(hops.sum()), 1), "first_done": round(float(dd[0]), 1),
                 "proc_us(ready->done)": q(proc), "done_by_level_us": done_by_level, "wait_us(start->ready)": q(wait),
                 "done_after_prev_level_us": q(lag), "start_after_prev_level_us": q(start_lag),
                 "ready_after_prev_level_us": q(np.array([t[i, 1] - prev_done[lv[i]] for i in np.nonzero(sel)[0]
                                                          if lv[i] in prev_done]))}
print(json.dumps(out, indent=1))
