"""Per-phase cycles of the segmented one-sweep sort (batched evaluation, config 5), PDNN_SORT_TRACE=1."""
import ctypes, os, sys
os.environ["PDNN_SORT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2008_08636_b200 import Graph, load_library
from synth import make_config, candidate_parts
w = make_config(5)
G = Graph(w.V, w.src, w.dst); G.set_costs(w.c, w.w)
B = int(os.environ.get("BS", "64"))
parts = torch.as_tensor(candidate_parts(w.seed, 0, B, w.V, w.n_pe, "uniform")).cuda()
G.eval_batch(parts, w.n_pe, w.mem, w.kind, w.cap_eff)
torch.cuda.synchronize()
lib = load_library()
buf = (ctypes.c_ulonglong * 16)()
lib.pdnn_debug_osort_trace(buf)
t = np.array(buf[:8], dtype=np.float64)
names = ["ticket->load issued", "load+ranks", "warp scan", "tile offsets+publish", "look-back", "smem reorder", "write runs", "clear+next ticket"]
tot = t.sum()
for n, x in zip(names, t):
    print(f"{n:24s} {x / tot * 100:5.1f}%")
