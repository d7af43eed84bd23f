"""World-size-2 gloo test of the batched-evaluation sharding + gather path
(CPU only).  Each rank evaluates its shard of candidates with the oracle (a
CPU stand-in for the per-rank GPU evaluator) and the result structs are
gathered with paper_2008_08636_b200.dist; every rank must end with the same
bytes as a single-process evaluation of all candidates."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B, q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import OracleGraph
    from paper_2008_08636_b200.dist import RESULT_BYTES, gather_results, shard_range
    from synth import candidate_parts, make_config

    w = make_config(1)
    og = OracleGraph(w.V, w.src, w.dst)
    b0, b1, per = shard_range(B, rank, world)
    parts = candidate_parts(w.seed, b0, b1, w.V, w.n_pe)
    res = og.eval_batch(w.c, w.w, w.mem, w.kind, w.n_pe, w.cap_eff, parts, n_threads=1)
    local = torch.zeros(per * RESULT_BYTES, dtype=torch.uint8)
    raw = torch.from_numpy(res.view(np.uint8).copy())
    local[: raw.numel()] = raw
    out = gather_results(local, B, world)
    q.put((rank, out.numpy().tobytes()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("B", [7, 8])
def test_gloo_shard_and_gather(B):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import OracleGraph
    from synth import candidate_parts, make_config

    w = make_config(1)
    og = OracleGraph(w.V, w.src, w.dst)
    ref = og.eval_batch(w.c, w.w, w.mem, w.kind, w.n_pe, w.cap_eff, candidate_parts(w.seed, 0, B, w.V, w.n_pe),
                        n_threads=2)
    assert got[0] == got[1] == ref.view(np.uint8).tobytes()


def test_shard_range_covers():
    from paper_2008_08636_b200.dist import shard_range

    for B in (0, 1, 5, 4096):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                b0, b1, per = shard_range(B, r, world)
                assert b1 - b0 <= per
                seen += list(range(b0, b1))
            assert seen == list(range(B))


def _bench_worker(rank, world, port, B, q):
    """bench.py's own shard_and_gather (the production batched path) on gloo,
    with the oracle standing in for the per-rank GPU evaluator."""
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from oracle import OracleGraph
    from paper_2008_08636_b200.dist import RESULT_BYTES
    from synth import candidate_parts, make_config

    w = make_config(1)
    og = OracleGraph(w.V, w.src, w.dst)

    def evaluate(b0, b1, per):
        local = torch.zeros(per * RESULT_BYTES, dtype=torch.uint8)
        if b1 > b0:
            res = og.eval_batch(w.c, w.w, w.mem, w.kind, w.n_pe, w.cap_eff,
                                candidate_parts(w.seed, b0, b1, w.V, w.n_pe), n_threads=1)
            raw = torch.from_numpy(res.view(np.uint8).copy())
            local[: raw.numel()] = raw
        return local

    out = bench.shard_and_gather(evaluate, B, rank, world)
    q.put((rank, out.numpy().tobytes()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("B", [1, 9])
def test_bench_shard_and_gather_gloo(B):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import OracleGraph
    from synth import candidate_parts, make_config

    w = make_config(1)
    og = OracleGraph(w.V, w.src, w.dst)
    ref = og.eval_batch(w.c, w.w, w.mem, w.kind, w.n_pe, w.cap_eff, candidate_parts(w.seed, 0, B, w.V, w.n_pe),
                        n_threads=2)
    assert got[0] == got[1] == ref.view(np.uint8).tobytes()
