#!/usr/bin/env python
"""bench.py -- the weighted-level sweep hot path of ParDNN (arXiv 2008.08636) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

One step (config 4 by default: the E3D-shaped 1.5M-node / 4.6M-edge DAG, 8 PEs)
is one pass of the hot path, through the C ABI:
  a6  pdnn_slice(K)             K slicing sweeps (tl+bl) + CP + removal
  a3/a4 pdnn_weighted_levels    placement-aware sweep under a P-way placement
  a5  pdnn_critical_path        CP of that placement
  a7  pdnn_memory_potential     memory tracker with st = tl under the placement
Graph construction (rows a1/a2, once per graph) and cost binding are outside
the timed region.  metric = (sweeps per step x 2|E|) / step time, in GTEPS.
The batched evaluation (row a8, config 5 = TRN graph x 4096 candidates) is
reported in the "batched" object.

Multi-GPU (torchrun, one rank per GPU): the single-graph step runs as
independent replicas (a single graph is never split: DESIGN.md "Multi-GPU"),
scaling "weak"; the batched candidates are sharded across ranks and the result
structs gathered with NCCL all_gather_into_tensor.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}
REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting",
           0x1: "gpu_idle", 0x10: "sync_boost", 0x100: "display_clock_setting"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=4096, help="candidates of config 5 per timed batch (all ranks)")
    ap.add_argument("--no-batch", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-shapes", action="store_true", help="skip the per-shape report (configs 2, 3, 6-9)")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    return dict(PEAKS_FALLBACK)


def host_info():
    cores = len(os.sched_getaffinity(0))
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return cores, model


# ------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, bus_id=None):
        self.proc = None
        self.bus_id = bus_id

    def __enter__(self):
        cmd = ["nvidia-smi", "--query-gpu=pci.bus_id,clocks.sm,clocks.max.sm,clocks_event_reasons.active",
               "--format=csv,noheader,nounits", "-lms", "100"]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.out = ""

    def summary(self):
        sm, mx, mask = [], [], 0
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 4:
                continue
            if self.bus_id and f[0].lower()[-12:] != self.bus_id.lower()[-12:]:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                mask |= int(f[3], 16)
            except ValueError:
                continue
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        reasons = sorted(n for b, n in REASONS.items() if mask & b and n != "gpu_idle")
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": reasons, "samples": len(sm)}


# ------------------------------------------------------------------ oracle (CPU baseline / reference arm)
def oracle_step(og, w, part, K):
    og.slice(w.c, w.w, K)
    tl, bl = og.weighted_levels(w.c, w.w, part)
    og.critical_path(w.c, w.w, part, tl, bl)
    og.memory(part, w.n_pe, w.mem, w.kind, tl, w.cap_eff)


def run_oracle(w, part, K, budget_s=None, steps=None, warmup=0):
    from oracle import OracleGraph

    og = OracleGraph(w.V, w.src, w.dst)
    for _ in range(warmup):
        oracle_step(og, w, part, K)
    n, t0 = 0, time.perf_counter()
    while True:
        oracle_step(og, w, part, K)
        n += 1
        dt = time.perf_counter() - t0
        if steps is not None and n >= steps:
            break
        if budget_s is not None and dt >= budget_s:
            break
    return n, dt


def spawn_ranks(n: int) -> int:
    """`--gpus N` without a launcher: re-run this script under torchrun with N
    ranks on this node (127.0.0.1 rendezvous) and return its exit code."""
    import socket

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1")))


def config_dict(name, w, D, K, sweeps, world):
    """The workload description both arms print (the driver compares them)."""
    return {"workload": name, "V": w.V, "E": w.E, "n_levels": D, "n_pe": w.n_pe, "K": K, "sweeps_per_step": sweeps,
            "seed": w.seed, "l2": "flushed between steps (256 MiB write, outside the per-step events); working set > L2",
            "parallelism": f"replicas x{world}" if world > 1 else "single GPU"}


def shard_and_gather(evaluate, B: int, rank: int, world: int):
    """Batched evaluation across ranks: rank r evaluates
    its contiguous shard [b0, b1) of the B candidates -- evaluate(b0, b1, per)
    returns its zero-padded uint8 [per * RESULT_BYTES] result structs -- and the
    structs of every rank are gathered (NCCL all_gather over NVLink; gloo in
    the CPU test).  Returns uint8 [B * RESULT_BYTES] on every rank, candidate order."""
    from paper_2008_08636_b200.dist import gather_results, shard_range

    b0, b1, per = shard_range(B, rank, world)
    return gather_results(evaluate(b0, b1, per), B, world)


# ------------------------------------------------------------------ main
def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    from synth import CONFIG_NAMES, candidate_parts, make_config

    w = make_config(args.config)
    K = max(w.K, 1)
    sweeps = K + 1
    part_np = candidate_parts(w.seed, 0, 1, w.V, w.n_pe, "refine")[0].astype(np.int32)

    if args.impl == "reference":
        if rank != 0:
            return
        cores, model = host_info()
        from oracle import OracleGraph

        D_ref = OracleGraph(w.V, w.src, w.dst).n_levels
        n, dt = run_oracle(w, part_np, K, steps=args.steps, warmup=args.warmup)
        v = n * sweeps * 2 * w.E / dt / 1e9
        line = {
            "impl": "reference", "metric": "tl+bl+CP sweep GTEPS", "value": v, "unit": "GTEPS",
            "n_gpus": 0, "steps": n, "warmup": args.warmup, "ms_per_step": dt / n * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic",
            "config": config_dict(CONFIG_NAMES[args.config], w, D_ref, K, sweeps, world),
            "cpu_baseline": {"value": v, "unit": "GTEPS", "cores": 1, "kind": "oracle",
                             "sample": f"{n} full steps of {CONFIG_NAMES[args.config]} (single-threaded C oracle, {model})"},
            "e2e": {"value": v, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line))
        return

    import torch
    import torch.distributed as dist

    if not torch.cuda.is_available() or torch.cuda.device_count() < (world if world > 1 else 1):
        raise SystemExit(f"bench.py: needs {max(world, 1)} CUDA device(s), found "
                         f"{torch.cuda.device_count() if torch.cuda.is_available() else 0}")
    if world > 1:
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local_rank if world > 1 else torch.cuda.current_device())
    torch.cuda.set_device(dev)
    from paper_2008_08636_b200 import EVAL_RESULT_DTYPE, Graph, launch_count, load_library

    lib = load_library()
    G = Graph(w.V, w.src, w.dst, device=dev)
    G.set_costs(w.c, w.w)
    ws = G.workspace()
    wsb = ws.numel()
    P = w.n_pe
    D = G.n_levels
    cap = max(D, 1)
    i32, i64 = torch.int32, torch.int64
    part = torch.as_tensor(part_np).to(dev)
    mem = torch.as_tensor(w.mem).to(dev)
    kind = torch.as_tensor(w.kind).to(dev)
    capeff = torch.as_tensor(w.cap_eff).to(dev)
    class Outs:  # the device outputs of one step (two sets for the pipelined e2e loop)
        def __init__(self):
            self.tl = torch.empty(w.V, dtype=i64, device=dev)
            self.bl = torch.empty(w.V, dtype=i64, device=dev)
            self.cps = torch.empty((K, cap), dtype=i32, device=dev)
            self.lens = torch.empty(K, dtype=i32, device=dev)
            self.Ls = torch.empty(K, dtype=i64, device=dev)
            self.hs = torch.empty(K, dtype=i64, device=dev)
            self.cp = torch.empty(cap, dtype=i32, device=dev)
            self.scal = torch.zeros(3, dtype=i64, device=dev)
            self.mpot = torch.empty(w.V, dtype=i64, device=dev)
            self.peak = torch.empty(P, dtype=i64, device=dev)
            self.ppos = torch.empty(P, dtype=i32, device=dev)
            self.fo = torch.empty(P, dtype=i32, device=dev)
            self.ob = torch.empty(P, dtype=i64, device=dev)

    outs0 = Outs()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    s = stream.cuda_stream

    def chk(rc, what):
        if rc != 0:
            raise RuntimeError(f"{what}: {rc} {lib.pdnn_last_error().decode()}")

    def step(ev=None, part_t=part, mem_t=mem, kind_t=kind, cap_t=capeff, o=outs0, st=stream):
        sp = st.cuda_stream
        if ev:
            ev[0].record(st)
        chk(lib.pdnn_slice(G.handle, None, None, K, cap, o.cps.data_ptr(), o.lens.data_ptr(), o.Ls.data_ptr(),
                           o.hs.data_ptr(), ws.data_ptr(), wsb, sp), "slice")
        if ev:
            ev[1].record(st)
        chk(lib.pdnn_weighted_levels(G.handle, None, None, part_t.data_ptr(), o.tl.data_ptr(), o.bl.data_ptr(),
                                     ws.data_ptr(), wsb, sp), "weighted_levels")
        if ev:
            ev[2].record(st)
        chk(lib.pdnn_critical_path(G.handle, None, None, part_t.data_ptr(), o.tl.data_ptr(), o.bl.data_ptr(),
                                   o.cp.data_ptr(), o.scal.data_ptr(), o.scal.data_ptr() + 8,
                                   o.scal.data_ptr() + 16, ws.data_ptr(), wsb, sp), "critical_path")
        if ev:
            ev[3].record(st)
        chk(lib.pdnn_memory_potential(G.handle, part_t.data_ptr(), P, mem_t.data_ptr(), kind_t.data_ptr(),
                                      o.tl.data_ptr(), cap_t.data_ptr(), o.mpot.data_ptr(), o.peak.data_ptr(),
                                      o.ppos.data_ptr(), o.fo.data_ptr(), o.ob.data_ptr(), None, ws.data_ptr(),
                                      wsb, sp), "memory_potential")
        if ev:
            ev[4].record(st)

    for _ in range(max(args.warmup, 0)):
        flush.zero_()
        step()
    torch.cuda.synchronize()

    # ---------------------------------------------------------------- timed region (device)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    bus = None
    try:
        pr = torch.cuda.get_device_properties(dev)
        bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
    except Exception:
        bus = None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # The same step captured once as a CUDA graph (one launch per step instead
    # of ~20 ctypes-driven ones); the headline is timed on its replays, the
    # per-call breakdown and the roofline on the eager calls.
    step_graph = None
    try:
        cs = torch.cuda.Stream(dev)
        cs.wait_stream(stream)
        g_ = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_, stream=cs):
            step(st=cs)
        stream.wait_stream(cs)
        step_graph = g_
        for _ in range(max(args.warmup, 0)):
            flush.zero_()
            step_graph.replay()
        torch.cuda.synchronize()
    except Exception:
        step_graph = None
        torch.cuda.synchronize()
    gevs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    l0 = launch_count()
    with ClockSampler(bus) as clk:
        t_wall = time.perf_counter()
        for k in range(args.steps):
            flush.zero_()                # L2 flush between steps, outside the step events
            step(evs[k])
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
        launches = launch_count() - l0
        if step_graph is not None:
            for k in range(args.steps):
                flush.zero_()
                gevs[k][0].record(stream)
                step_graph.replay()
                gevs[k][1].record(stream)
            torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    seg = np.array([[evs[k][j].elapsed_time(evs[k][j + 1]) for j in range(4)] for k in range(args.steps)])
    step_ms = seg.sum(axis=1)
    eager_ms_per_step = float(step_ms.sum()) / args.steps
    total_ms = float(step_ms.sum())
    if step_graph is not None:
        total_ms = float(sum(gevs[k][0].elapsed_time(gevs[k][1]) for k in range(args.steps)))
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    edges_per_step = sweeps * 2 * w.E
    value = world * args.steps * edges_per_step / (total_ms / 1e3) / 1e9

    # roofline of the dominant kernel: the placement-aware sweep launch
    pk = peaks()
    sweep_ms = float(np.mean(seg[:, 1]))
    alg_bytes = 24 * w.E + 48 * w.V        # SURVEY.md 8(d) compulsory bytes per sweep
    achieved = alg_bytes / (sweep_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(CONFIG_NAMES[args.config], {}).get("k_sweep")
        except Exception:
            traffic = None

    # ---------------------------------------------------------------- e2e (host buffers)
    # Every step copies its input -- the placement being evaluated and the PE
    # capacities -- from pinned host memory and reads ALL its results back to
    # pinned host memory: tl / bl of the placement, M_pot, the placement CP and
    # the K slicing CPs, L / hash / per-PE summaries.  The
    # per-node profiles (comp / comm costs, mem, kinds) are graph attributes:
    # uploaded once with the graph (pdnn_graph_set_costs; mem / kind tensors),
    # as a refinement loop evaluating placement after placement would.  The
    # loop is a standard two-deep pipeline: step k's H2D (copy stream) and step
    # k-1's D2H (a second copy stream) overlap step k-1's / k's kernels;
    # double-buffered device inputs and outputs, events order every reuse.
    h_part = torch.as_tensor(part_np).pin_memory()
    h_cap = torch.as_tensor(w.cap_eff).pin_memory()
    n_small = 3 + 3 * P + K * 3
    bufs = []
    for _ in range(2):
        b = {"in": [torch.empty_like(x, device=dev) for x in (h_part, h_cap)],
             "out": outs0 if not bufs else Outs(),
             "small": torch.empty(n_small, dtype=i64, device=dev),
             "h_mpot": torch.empty(w.V, dtype=i64).pin_memory(),
             "h_tl": torch.empty(w.V, dtype=i64).pin_memory(),
             "h_bl": torch.empty(w.V, dtype=i64).pin_memory(),
             "h_cps": torch.empty((K, cap), dtype=i32).pin_memory(),
             "h_cp": torch.empty(cap, dtype=i32).pin_memory(),
             "h_small": torch.empty(n_small, dtype=i64).pin_memory(),
             "h2d_done": torch.cuda.Event(), "comp_done": torch.cuda.Event(), "d2h_done": torch.cuda.Event()}
        bufs.append(b)
    h2d = sum(x.numel() * x.element_size() for x in (h_part, h_cap))
    d2h = sum(bufs[0][k].numel() * bufs[0][k].element_size() for k in ("h_mpot", "h_tl", "h_bl", "h_cps", "h_cp", "h_small"))
    s_h2d = torch.cuda.Stream(dev)
    s_d2h = torch.cuda.Stream(dev)

    # The step's launches (every library call of the step and the result
    # packing) are captured once per buffer set into a CUDA graph, so the
    # host issues one graph launch per step instead of ~20 launches through
    # ctypes; without graph support the loop issues the calls eagerly.
    def compute(b, st):
        o = b["out"]
        step(None, b["in"][0], mem, kind, b["in"][1], o=o, st=st)   # mem / kind: device-resident graph attributes
        torch.cat([o.scal, o.peak, o.ob, o.ppos.to(i64), o.Ls, o.hs, o.lens.to(i64)], out=b["small"])

    graphs, graph_note = [None, None], "eager"
    try:
        cs = torch.cuda.Stream(dev)
        for idx in range(2):
            cs.wait_stream(stream)
            g_ = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_, stream=cs):
                compute(bufs[idx], cs)
            graphs[idx] = g_
        stream.wait_stream(cs)
        graph_note = "cuda graph per step"
    except Exception as ex:   # capture unsupported: eager launches
        graphs, graph_note = [None, None], "eager (graph capture failed: " + str(ex).splitlines()[0][:120] + ")"
        torch.cuda.synchronize()

    def e2e_step(k):
        b = bufs[k % 2]
        o = b["out"]
        with torch.cuda.stream(s_h2d):
            s_h2d.wait_event(b["comp_done"])    # step k-2 has consumed these inputs
            for d_x, h_x in zip(b["in"], (h_part, h_cap)):
                d_x.copy_(h_x, non_blocking=True)
            b["h2d_done"].record(s_h2d)
        stream.wait_event(b["h2d_done"])
        stream.wait_event(b["d2h_done"])        # step k-2's results are on the host
        if graphs[k % 2] is not None:
            with torch.cuda.stream(stream):
                graphs[k % 2].replay()
        else:
            compute(b, stream)
        b["comp_done"].record(stream)
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_event(b["comp_done"])
            b["h_mpot"].copy_(o.mpot, non_blocking=True)
            b["h_tl"].copy_(o.tl, non_blocking=True)
            b["h_bl"].copy_(o.bl, non_blocking=True)
            b["h_cps"].copy_(o.cps, non_blocking=True)
            b["h_cp"].copy_(o.cp, non_blocking=True)
            b["h_small"].copy_(b["small"], non_blocking=True)
            b["d2h_done"].record(s_d2h)

    for k in range(2):
        e2e_step(k)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(args.steps):
        e2e_step(k)
    torch.cuda.synchronize()                    # every result of every step is on the host
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = world * args.steps * edges_per_step / e2e_s / 1e9
    # the last step's host copy agrees with the device result (the pipeline moved real data)
    last = bufs[(args.steps - 1) % 2]
    assert torch.equal(last["h_mpot"], last["out"].mpot.cpu()), "e2e pipeline: M_pot copy mismatch"
    assert torch.equal(last["h_tl"], last["out"].tl.cpu()), "e2e pipeline: tl copy mismatch"

    # ---------------------------------------------------------------- batched evaluation (config 5)
    batched = None
    if not args.no_batch and args.batch > 0:
        from paper_2008_08636_b200.dist import RESULT_BYTES, shard_range

        w5 = make_config(5)
        G5 = Graph(w5.V, w5.src, w5.dst, device=dev)
        G5.set_costs(w5.c, w5.w)
        B = args.batch
        b0, b1, per = shard_range(B, rank, world)
        parts5 = torch.as_tensor(candidate_parts(w5.seed, b0, b1, w5.V, w5.n_pe, "uniform")).to(dev)
        mem5, kind5, cap5 = (torch.as_tensor(x).to(dev) for x in (w5.mem, w5.kind, w5.cap_eff))
        out5 = torch.zeros(per * RESULT_BYTES, dtype=torch.uint8, device=dev)

        def evaluate(e0, e1, n_per, parts=parts5):
            if e1 > e0:
                G5.eval_batch(parts, w5.n_pe, mem5, kind5, cap5, out=out5)
            return out5

        shard_and_gather(evaluate, B, rank, world)   # warm-up (also sizes the workspace)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        reps = 3
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):   # each rep: evaluate this rank's shard, gather every rank's results
            res = shard_and_gather(evaluate, B, rank, world)
        e1.record(stream)
        torch.cuda.synchronize()
        bt = e0.elapsed_time(e1) / reps
        if world > 1:
            t = torch.tensor([bt], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            bt = float(t.item())
        assert res.numel() == B * RESULT_BYTES
        # the "refinement trials" distribution (a base placement with ~1% of the
        # nodes re-labelled per candidate)
        parts_r = torch.as_tensor(candidate_parts(w5.seed, b0, b1, w5.V, w5.n_pe, "refine")).to(dev)
        shard_and_gather(lambda e0_, e1_, n_: evaluate(e0_, e1_, n_, parts=parts_r), B, rank, world)
        torch.cuda.synchronize()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        for _ in range(reps):
            shard_and_gather(lambda e0_, e1_, n_: evaluate(e0_, e1_, n_, parts=parts_r), B, rank, world)
        r1.record(stream)
        torch.cuda.synchronize()
        bt_r = r0.elapsed_time(r1) / reps
        if world > 1:
            t = torch.tensor([bt_r], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            bt_r = float(t.item())
        del parts_r
        # one GPU: the time of the 8-GPU shard (B / 8 candidates) -> the
        # projected 8-GPU strong-scaling ratio T(B) / T(B / 8)
        proj = None
        if world == 1 and B >= 8:
            n8 = (B + 7) // 8
            sub = parts5[:n8]
            G5.eval_batch(sub, w5.n_pe, mem5, kind5, cap5, out=out5)
            torch.cuda.synchronize()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            for _ in range(reps):
                G5.eval_batch(sub, w5.n_pe, mem5, kind5, cap5, out=out5)
            f1.record(stream)
            torch.cuda.synchronize()
            t8 = f0.elapsed_time(f1) / reps
            proj = {"shard_candidates": n8, "shard_ms": t8, "projected_8gpu_scaling": bt / t8}
        pk5 = peaks()
        alg5 = 23 * w5.E + 35 * w5.V          # sweep 18E+26V + memory 5E+9V per candidate
        ach5 = B * alg5 / (bt / 1e3) / 1e9
        batched = {"metric": "batched partition evals/s", "value": B / (bt / 1e3), "unit": "evals/s",
                   "per_gpu_evals_s": B / (bt / 1e3) / world, "n_gpus": world,
                   "candidates": B, "of": 4096, "workload": CONFIG_NAMES[5], "V": w5.V, "E": w5.E,
                   "n_levels": G5.n_levels, "ms": bt, "reps": reps, "scaling": "strong",
                   "distribution": "uniform iid labels (value); refinement trials in refine_*",
                   "refine_evals_s": B / (bt_r / 1e3), "refine_ms": bt_r,
                   "gather": ("dist.gather_results: NCCL all_gather_into_tensor" if world > 1 else None),
                   "roofline": {"bound": "hbm", "achieved": ach5, "peak": pk5.get("hbm_gbs"), "unit": "GB/s",
                                "frac": ach5 / pk5.get("hbm_gbs"), "alg_bytes_per_candidate": alg5,
                                "peak_source": pk5.get("source")},
                   "projection_1gpu": proj}
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            # the oracle on every host core (one candidate per thread), a bounded sample
            from oracle import OracleGraph

            cores, model = host_info()
            og5 = OracleGraph(w5.V, w5.src, w5.dst)
            nc = 32 * cores
            sp = candidate_parts(w5.seed, 0, nc, w5.V, w5.n_pe, "uniform")
            t0 = time.perf_counter()
            og5.eval_batch(w5.c, w5.w, w5.mem, w5.kind, w5.n_pe, w5.cap_eff, sp, n_threads=cores)
            dtc = time.perf_counter() - t0
            batched["cpu_baseline"] = {"value": nc / dtc, "unit": "evals/s", "cores": cores, "kind": "oracle",
                                       "sample": f"{nc} candidates of {CONFIG_NAMES[5]} ({dtc:.1f} s), C oracle, "
                                                 f"one candidate per thread on {cores} threads ({model})"}

    # ---------------------------------------------------------------- the other graph shapes
    # The same single-graph step on the other shapes north_star names (Word-RNN,
    # TRN, Char-CRN, WRN) and on C4's node set at D = 256 and at E3D's degree of
    # parallelism: GTEPS, the placement sweep's HBM fraction, depth D, DoP and
    # CCR as generated (Table 5 targets in DESIGN.md).  Eager calls, L2 flushed.
    shapes = None
    if not args.no_shapes and rank == 0:
        shapes = {}
        for n in (2, 3, 6, 7, 8, 9):
            ws_ = make_config(n)
            Gs = Graph(ws_.V, ws_.src, ws_.dst, device=dev)
            Gs.set_costs(ws_.c, ws_.w)
            ps = torch.as_tensor(candidate_parts(ws_.seed, 0, 1, ws_.V, ws_.n_pe, "refine")[0].astype(np.int32)).to(dev)
            ms_, ks_, cs_ = (torch.as_tensor(x).to(dev) for x in (ws_.mem, ws_.kind, ws_.cap_eff))
            Ks = max(ws_.K, 1)

            def one_step():
                Gs.slice(Ks)
                tl_, bl_ = Gs.weighted_levels(ps)
                Gs.critical_path(tl_, bl_, ps)
                Gs.memory_potential(ps, ws_.n_pe, ms_, ks_, tl_, cs_)

            one_step()
            z = torch.zeros(ws_.V, dtype=torch.int32, device=dev)
            tl0, bl0 = Gs.weighted_levels(z)           # all on one PE: the computation-only CP
            L0 = int((tl0 + bl0).max().item())
            # median of 5 eager reps: robust to a host-side stall between the
            # event records (a full bench run once showed one C8 rep 100x slow
            # right after the oracle's all-core baseline; 100 isolated reps did not)
            reps = 5
            seg_r = []
            rep_wl = []
            for _ in range(reps):
                flush.zero_()
                ev_ = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
                ev_[0].record(stream)
                Gs.slice(Ks)
                ev_[1].record(stream)
                tl_, bl_ = Gs.weighted_levels(ps)
                ev_[2].record(stream)
                Gs.critical_path(tl_, bl_, ps)
                ev_[3].record(stream)
                Gs.memory_potential(ps, ws_.n_pe, ms_, ks_, tl_, cs_)
                ev_[4].record(stream)
                torch.cuda.synchronize()
                seg_r.append([ev_[j].elapsed_time(ev_[j + 1]) for j in range(4)])
                rep_wl.append(round(ev_[1].elapsed_time(ev_[2]), 4))
            seg_r = np.array(seg_r)
            seg_s = seg_r[np.argsort(seg_r.sum(axis=1))[reps // 2]]    # the median rep (by step time)
            step = float(seg_s.sum())
            sw = float(np.median(seg_r[:, 1]))
            alg_s = 24 * ws_.E + 48 * ws_.V
            shapes[CONFIG_NAMES[n]] = {
                "V": ws_.V, "E": ws_.E, "D": Gs.n_levels, "n_pe": ws_.n_pe, "K": Ks,
                "dop": float(ws_.c.sum()) / max(L0, 1), "ccr": float(ws_.w.sum()) / max(float(ws_.c.sum()), 1.0),
                "ms_per_step": step, "GTEPS": (Ks + 1) * 2 * ws_.E / (step / 1e3) / 1e9,
                "sweep_ms": sw, "sweep_hbm_frac": alg_s / (sw / 1e3) / 1e9 / peaks().get("hbm_gbs"),
                "breakdown_ms": {"slice": float(seg_s[0]), "weighted_levels": float(seg_s[1]),
                                 "critical_path": float(seg_s[2]), "memory": float(seg_s[3])},
                "us_per_level_pair": sw * 1e3 / max(Gs.n_levels, 1), "weighted_levels_reps_ms": rep_wl}
            del Gs
            torch.cuda.empty_cache()

    # ---------------------------------------------------------------- CPU baseline (oracle)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores, model = host_info()
        n, dt = run_oracle(w, part_np, K, budget_s=args.cpu_seconds)
        cpu = {"value": n * edges_per_step / dt / 1e9, "unit": "GTEPS", "cores": 1, "kind": "oracle",
               "sample": f"{n} full steps ({dt:.1f} s) of {CONFIG_NAMES[args.config]}, single-threaded C oracle "
                         f"on {model} ({cores} host cores available)"}

    if rank == 0:
        line = {
            "metric": "tl+bl+CP sweep GTEPS", "value": value, "unit": "GTEPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": config_dict(CONFIG_NAMES[args.config], w, D, K, sweeps, world),
            "breakdown_ms": {"slice": float(np.mean(seg[:, 0])), "weighted_levels": sweep_ms,
                             "critical_path": float(np.mean(seg[:, 2])), "memory": float(np.mean(seg[:, 3]))},
            "roofline": {"kernel": "k_sweep<1> (pdnn_weighted_levels: one launch, its in-kernel label pass included; events around the call, so achieved is a lower bound)",
                         "bound": "hbm", "achieved": achieved,
                         "peak": pk.get("hbm_gbs"), "unit": "GB/s", "frac": achieved / pk.get("hbm_gbs"),
                         "traffic": traffic, "alg_bytes": alg_bytes, "peak_source": pk.get("source")},
            "gpu_launches": int(launches),
            "e2e": {"value": e2e_value, "unit": "GTEPS", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "pipeline": "H2D and D2H on two copy streams, double-buffered, overlapped with the kernels; " + graph_note},
            "clocks": clk.summary(),
            "wall_ms_per_step_incl_flush": t_wall / args.steps * 1e3,
            "timing": ("CUDA-graph replay of the step (one graph launch per step), events around each replay; "
                       "breakdown_ms / roofline from the same step issued eagerly" if step_graph is not None
                       else "eager library calls, events around each call"),
            "eager_ms_per_step": eager_ms_per_step,
            "batched": batched,
            "shapes": shapes,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
