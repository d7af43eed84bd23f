"""Per-phase timeline of the chunked visit-order sort on config 4 (PDNN_SORT_TRACE=1)."""
import ctypes, os, sys
os.environ["PDNN_SORT_TRACE"] = "1"
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
buf = (ctypes.c_ulonglong * 128)()
lib.pdnn_debug_sort_trace(buf)
t = np.array(buf[:], dtype=np.int64)
for c, off in (("cta0", 0), ("ctaLast", 64)):
    base = t[off]
    print(c, [[int(t[off + p * 10 + k] - base) if t[off + p * 10 + k] else None for k in range(9)] for p in range(5)])
