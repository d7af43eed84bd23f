"""Time pdnn_build_csr (graph construction incl. Kahn levels) per config, and
the oracle's build on this host."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
if os.environ.get("PDNN_BUILD_TRACE"):   # per-phase host times on stderr (debug library)
    from paper_2008_08636_b200 import _binding, build
    _binding.load_library(build.build(debug_knobs=True))
from paper_2008_08636_b200 import Graph
from synth import make_config
from oracle import OracleGraph
for cfg in os.environ.get("CFGS", "2,3,7").split(","):
    w = make_config(int(cfg))
    src, dst = torch.as_tensor(w.src).cuda(), torch.as_tensor(w.dst).cuda()
    Graph(w.V, src, dst); torch.cuda.synchronize()
    t = time.perf_counter(); G = Graph(w.V, src, dst); torch.cuda.synchronize(); tg = time.perf_counter() - t
    t = time.perf_counter(); og = OracleGraph(w.V, w.src, w.dst); to = time.perf_counter() - t
    assert G.n_levels == og.n_levels
    print(json.dumps({"cfg": cfg, "V": w.V, "D": G.n_levels, "gpu_build_ms": round(tg * 1e3, 2),
                      "oracle_build_ms": round(to * 1e3, 2)}), flush=True)
