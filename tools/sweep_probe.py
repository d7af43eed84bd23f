"""Time the sweep alone on a config and report poll statistics (debug tool)."""
import os, sys, json, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import make_config, candidate_parts
from paper_2008_08636_b200 import Graph
cfg = os.environ.get("CFG", "4")
if cfg == "chain":
    import types
    n = 20000
    rng = np.random.default_rng(0)
    w = types.SimpleNamespace(V=n, src=np.arange(n - 1, dtype=np.int32), dst=np.arange(1, n, dtype=np.int32),
                              c=rng.integers(0, 1000, n), w=rng.integers(0, 1000, n - 1), seed=1, n_pe=4)
else:
    w = make_config(int(cfg))
G = Graph(w.V, w.src, w.dst); G.set_costs(w.c, w.w)
part = torch.as_tensor(candidate_parts(w.seed, 0, 1, w.V, w.n_pe, "refine")[0].astype(np.int32)).cuda()
ws = G.workspace()
for _ in range(3): G.weighted_levels(part)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    ws[80:144].zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); G.weighted_levels(part); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
misc = ws[80:144].cpu().numpy().view(np.uint64)
print(json.dumps({"cfg": cfg, "sleep": os.environ.get("PDNN_POLL_SLEEP_NS"), "ms_med": float(np.median(ts)),
      "ms_min": float(min(ts)), "spins_per_warp": float(misc[0]) / max(1, misc[2]), "busy_us_per_warp": float(misc[1]) / max(1, misc[2]) / 1965.0,
      "warps": int(misc[2]), "tma_wait_us_per_warp": float(misc[3]) / max(1, misc[2]) / 1965.0, "proc_us_per_warp": float(misc[4]) / max(1, misc[2]) / 1965.0,
      "split_us_per_warp": float(misc[5]) / max(1, misc[2]) / 1965.0, "relax_us_per_warp": float(misc[6]) / max(1, misc[2]) / 1965.0, "n_items": None, "D": G.n_levels}))
