"""pdnn_refine phase times (debug library, PDNN_REFINE_TRACE=1 on stderr)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PDNN_REFINE_TRACE"] = "1"
import torch
from paper_2008_08636_b200 import _binding, build
_binding.load_library(build.build(debug_knobs=True, variant=os.environ.get("VARIANT", ""),
                                  defines=[d for d in os.environ.get("DEFS", "").split() if d]))
from paper_2008_08636_b200 import Graph
from synth import make_config
for n in [int(x) for x in sys.argv[1:]] or [2, 3]:
    w = make_config(n)
    G = Graph(w.V, w.src, w.dst); G.set_costs(w.c, w.w)
    cof, mem, off, nc = G.slice_clusters(w.K)
    nc = int(nc.item())
    p0, _ = G.lflam(cof, mem, off, nc, w.K)
    torch.cuda.synchronize()
    print("config", n, flush=True)
    part, log, L = G.refine(cof, mem, off, nc, w.K, p0)
    torch.cuda.synchronize()
    import hashlib
    print("log", len(log), hashlib.sha1(log.tobytes()).hexdigest()[:12], "L", L, flush=True)
