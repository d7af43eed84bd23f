"""Per-tile timeline of the single-pass memory scan on config 4 (PDNN_SCAN_TRACE=1)."""
import ctypes, os, sys
os.environ["PDNN_SCAN_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2008_08636_b200 import Graph, load_library
from synth import make_config, candidate_parts
w = make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
G = Graph(w.V, w.src, w.dst, device="cuda:0"); G.set_costs(w.c, w.w)
part = candidate_parts(w.seed, 0, 1, w.V, w.n_pe)[0].astype(np.int32)
tl, bl = G.weighted_levels(part)
for _ in range(3):
    G.memory_potential(part, w.n_pe, w.mem, w.kind, tl, w.cap_eff)
torch.cuda.synchronize()
lib = load_library()
buf = (ctypes.c_ulonglong * 16384)()
lib.pdnn_debug_scan_trace(buf)
t = np.array(buf[:], dtype=np.int64).reshape(-1, 4)
n = (w.V + 2047) // 2048
t = t[:n]
t0 = t[:, 0].min()
t = (t - t0) / 1000.0
print("tiles", n, "end", t[:, 3].max())
print("local work (start->published) us: median", np.median(t[:, 1] - t[:, 0]), "max", (t[:, 1] - t[:, 0]).max())
print("look-back us: median", np.median(t[:, 2] - t[:, 1]), "max", (t[:, 2] - t[:, 1]).max())
print("emit us: median", np.median(t[:, 3] - t[:, 2]), "max", (t[:, 3] - t[:, 2]).max())
for i in list(range(0, n, max(1, n // 24))) + [n - 1]:
    print(i, np.round(t[i], 2))
