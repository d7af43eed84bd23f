"""One C4 (CFG) placement sweep through the debug library, for ncu:
    VARIANT=_s2 DEFS=... PDNN_SWEEP_NOWAIT=1 ncu -k regex:k_sweep -s 3 -c 1 python tools/prof_sweep.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2008_08636_b200 import _binding, build
_defs = [d for d in os.environ.get("DEFS", "").split() if d]
_binding.load_library(build.build(debug_knobs=True, variant=os.environ.get("VARIANT", ""), defines=_defs))
from paper_2008_08636_b200 import Graph
from synth import make_config, candidate_parts
w = make_config(int(os.environ.get("CFG", "4")))
G = Graph(w.V, w.src, w.dst); G.set_costs(w.c, w.w)
part = torch.as_tensor(candidate_parts(w.seed, 0, 1, w.V, w.n_pe, "refine")[0].astype(np.int32)).cuda()
for _ in range(4):
    G.weighted_levels(part)
torch.cuda.synchronize()
