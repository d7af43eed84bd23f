"""Single-placement scheduler-emulator timing (NEXT row N1): pdnn_emulate beside
the oracle's or_emulate.  Usage: python tools/emulate_probe.py [config ...]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import OracleGraph
from paper_2008_08636_b200 import Graph
from synth import candidate_parts, make_config
for n in [int(x) for x in sys.argv[1:]] or [2, 3, 4]:
    w = make_config(n)
    G = Graph(w.V, w.src, w.dst); G.set_costs(w.c, w.w)
    part = candidate_parts(w.seed, 0, 1, w.V, w.n_pe, "uniform")[0].astype(np.int32)
    G.emulate(part, w.n_pe); torch.cuda.synchronize()
    t = time.perf_counter(); st, ft, mk = G.emulate(part, w.n_pe); torch.cuda.synchronize(); tg = time.perf_counter() - t
    og = OracleGraph(w.V, w.src, w.dst)
    t = time.perf_counter(); st_o, ft_o, mk_o, q = og.emulate(w.c, w.w, part, w.n_pe); to = time.perf_counter() - t
    print(json.dumps({"config": w.name, "V": w.V, "max_queue": int(q), "gpu_s": round(tg, 4), "oracle_s": round(to, 4),
                      "identical": bool(np.array_equal(st.cpu().numpy(), st_o) and int(mk.item()) == mk_o)}), flush=True)
