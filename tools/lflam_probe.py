"""LFLAM timing probe (NEXT row N4): pdnn_lflam (CUDA events, after a
warm-up call, clusters from pdnn_slice_clusters) beside the oracle's or_lflam
on the same clusters.  Usage: python tools/lflam_probe.py [config ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import OracleGraph  # noqa: E402
from paper_2008_08636_b200 import Graph, _binding, build  # noqa: E402

STATS = os.environ.get("LFLAM_STATS") == "1"     # debug-knob build: decisions evaluated / passes
if STATS:
    _binding.load_library(build.build(debug_knobs=True))
from synth import make_config  # noqa: E402

out = []
for n in [int(x) for x in sys.argv[1:]] or [2, 6, 3, 7, 4]:
    w = make_config(n)
    G = Graph(w.V, w.src, w.dst)
    G.set_costs(w.c, w.w)
    cof, mem, off, nc = G.slice_clusters(w.K)
    nc = int(nc.item())
    G.lflam(cof, mem, off, nc, w.K)                  # warm-up (workspace, smem attribute)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        part, log = G.lflam(cof, mem, off, nc, w.K)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    stats = None
    if STATS:
        import ctypes
        buf = (ctypes.c_uint64 * 2)()
        lib = _binding.load_library()
        lib.pdnn_debug_lflam_stats.argtypes = [ctypes.c_void_p] * 3
        ws = G.workspace(_binding.PDNN_OP_LFLAM, 0)
        lib.pdnn_debug_lflam_stats(G._h, ctypes.c_void_p(ws.data_ptr()), buf)
        stats = [int(buf[0]), int(buf[1])]
    og = OracleGraph(w.V, w.src, w.dst)
    cof_h, mem_h, off_h = cof.cpu().numpy(), mem.cpu().numpy(), off.cpu().numpy()[: nc + 1]
    cl = [mem_h[off_h[i]:off_h[i + 1]] for i in range(nc)]
    t = time.perf_counter()
    part_o, log_o = og.lflam(w.c, w.w, cof_h, cl, w.K)
    t_or = time.perf_counter() - t
    same = bool(np.array_equal(part.cpu().numpy(), part_o) and np.array_equal(log.cpu().numpy(), log_o))
    r = {"config": w.name, "V": w.V, "D": int(og.levels().max()) + 1, "clusters": nc, "decisions": len(log_o),
         "lookahead": int((log_o[:, 1] == 0).sum()), "gpu_ms": round(min(ts), 3), "oracle_ms": round(1e3 * t_or, 1),
         "identical": same, "evaluations_passes": stats}
    print(json.dumps(r), flush=True)
    out.append(r)
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/lflam_probe.json", "w") as f:
    json.dump(out, f, indent=1)
