"""Build (and drop) many tiny random DAGs back to back, hunting an
intermittent stall in pdnn_build_csr.  A watchdog thread reports the
iteration and exits the process if one build takes more than 20 s."""
import os, sys, threading, time, faulthandler
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2008_08636_b200 import Graph
from synth import tiny_random_dag
state = {"i": -1, "t": time.time(), "what": ""}
def watchdog():
    while True:
        time.sleep(2)
        if time.time() - state["t"] > 20:
            print("STALL at iteration", state["i"], state["what"], flush=True)
            faulthandler.dump_traceback()
            os._exit(3)
threading.Thread(target=watchdog, daemon=True).start()
rng = np.random.default_rng(int(os.environ.get("SEED", "5")))
N = int(os.environ.get("N", "3000"))
for i in range(N):
    n = int(rng.integers(3, 40))
    s, d = tiny_random_dag(rng, n, float(rng.uniform(0.1, 0.6)))
    state.update(i=i, t=time.time(), what=f"n={n} E={s.size}")
    G = Graph(n, s, d)
    if os.environ.get("WORK"):
        c, w = rng.integers(0, 5, n), rng.integers(0, 5, s.size)
        G.set_costs(c, w)
        G.slice_clusters(2)
    del G
torch.cuda.synchronize()
print("ok", N, flush=True)
