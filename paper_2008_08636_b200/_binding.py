"""ctypes binding of libpdnn.so (the C ABI in include/pdnn.h).

Argument marshalling only: every step of the weighted-level sweep, CP
extraction, memory scan and batched evaluation runs in the library's sm_100a
kernels.  PyTorch provides device memory and the stream.  There is no CPU
fallback: if the library or a CUDA device is missing, every call raises.

The module-level functions keep the C names (``pdnn_build_csr`` ...) and take
torch tensors; :class:`Graph` wraps a graph handle plus its workspace.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpdnn.so")

PDNN_REMOVED = -1
PDNN_UNASSIGNED = -2
PDNN_MAX_PE = 16
PDNN_KIND_NORMAL, PDNN_KIND_RESIDUAL, PDNN_KIND_REFERENCE = 0, 1, 2
PDNN_EDGE_ORDER_CANONICAL, PDNN_EDGE_ORDER_INPUT = 0, 1
PDNN_OP_WEIGHTED_LEVELS, PDNN_OP_CRITICAL_PATH, PDNN_OP_SLICE, PDNN_OP_MEMORY, PDNN_OP_EVAL_BATCH = 1, 2, 3, 4, 5
PDNN_OP_EMULATE, PDNN_OP_EVAL_BATCH_EMULATED, PDNN_OP_SLICE_CLUSTERS, PDNN_OP_RESOLVE_OVERFLOW = 6, 7, 8, 9
PDNN_OP_LFLAM = 10
PDNN_OP_REFINE = 11
PDNN_SCHEDULE_LEVEL, PDNN_SCHEDULE_EMULATED = 0, 1

EXPORTS = (
    "pdnn_build_csr", "pdnn_graph_free", "pdnn_graph_query", "pdnn_graph_levels",
    "pdnn_graph_set_costs", "pdnn_workspace_bytes", "pdnn_workspace_init",
    "pdnn_weighted_levels", "pdnn_critical_path", "pdnn_slice", "pdnn_memory_potential",
    "pdnn_eval_batch", "pdnn_emulate", "pdnn_validate", "pdnn_slice_clusters", "pdnn_criticality",
    "pdnn_resolve_overflow", "pdnn_lflam", "pdnn_refine",
    "pdnn_status_string", "pdnn_last_error", "pdnn_launch_count",
)

# pdnn_eval_result, 432 bytes (include/pdnn.h)
EVAL_RESULT_DTYPE = np.dtype(
    [
        ("L", "<i8"), ("cut_comm", "<i8"), ("cp_hash", "<u8"),
        ("cp_len", "<i4"), ("cp_start", "<i4"), ("cp_end", "<i4"), ("overflow_mask", "<i4"),
        ("peak", "<i8", (PDNN_MAX_PE,)), ("over_bytes", "<i8", (PDNN_MAX_PE,)),
        ("peak_pos", "<i4", (PDNN_MAX_PE,)), ("first_over_pos", "<i4", (PDNN_MAX_PE,)),
        ("makespan", "<i8"),
    ]
)
assert EVAL_RESULT_DTYPE.itemsize == 432


class PdnnError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        self.status = status
        self.name = _STATUS.get(status, str(status))
        super().__init__(f"{where}: {self.name} ({detail})")


_STATUS = {0: "PDNN_OK", -1: "PDNN_EINVAL", -2: "PDNN_ECYCLE", -3: "PDNN_ENOMEM", -4: "PDNN_ECUDA",
           -5: "PDNN_EOVERFLOW", -6: "PDNN_EWORKSPACE"}

_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load libpdnn.so (raises if it is missing: there is no fallback).
    PDNN_DEBUG_LIB=<path> (diagnostics only) loads a debug build instead."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if path == LIB_PATH and os.environ.get("PDNN_DEBUG_LIB"):
            path = os.environ["PDNN_DEBUG_LIB"]
        if not os.path.exists(path):
            raise RuntimeError(f"{path} not built; run `python -m paper_2008_08636_b200.build`")
        lib = C.CDLL(path)
        P, I32, I64 = C.c_void_p, C.c_int32, C.c_int64
        sig = {
            "pdnn_build_csr": ([I32, I64, P, P, P, P, C.POINTER(P)], C.c_int),
            "pdnn_graph_free": ([P], None),
            "pdnn_graph_query": ([P, P, P, P, P, P], C.c_int),
            "pdnn_graph_levels": ([P, P, P], C.c_int),
            "pdnn_graph_set_costs": ([P, P, P, C.c_int, P], C.c_int),
            "pdnn_workspace_bytes": ([P, C.c_int, I32], C.c_size_t),
            "pdnn_workspace_init": ([P, C.c_size_t, P], C.c_int),
            "pdnn_weighted_levels": ([P, P, P, P, P, P, P, C.c_size_t, P], C.c_int),
            "pdnn_critical_path": ([P] * 10 + [P, C.c_size_t, P], C.c_int),
            "pdnn_slice": ([P, P, P, I32, I32, P, P, P, P, P, C.c_size_t, P], C.c_int),
            "pdnn_memory_potential": ([P, P, I32] + [P] * 11 + [C.c_size_t, P], C.c_int),
            "pdnn_eval_batch": ([P, P, P, P, P, I32, P, I32, P, P, I32, P, C.c_size_t, P], C.c_int),
            "pdnn_emulate": ([P, P, P, P, I32, P, P, P, P, C.c_size_t, P], C.c_int),
            "pdnn_validate": ([P, P, P, P, I32, P, P, P, P], C.c_int),
            "pdnn_slice_clusters": ([P, P, P, I32, P, P, P, P, P, C.c_size_t, P], C.c_int),
            "pdnn_criticality": ([P, P, P, P, I32, P, P, C.c_size_t, P], C.c_int),
            "pdnn_resolve_overflow": ([P, P, P, P, P, I32, P, P, I32, P, P, P, P, C.c_size_t, P], C.c_int),
            "pdnn_lflam": ([P, P, P, P, P, P, I32, I32, P, P, P, P, C.c_size_t, P], C.c_int),
            "pdnn_refine": ([P, P, P, P, P, P, I32, I32, I32, I32, P, P, I32, P, P, P, C.c_size_t, P], C.c_int),
            "pdnn_status_string": ([C.c_int], C.c_char_p),
            "pdnn_last_error": ([], C.c_char_p),
            "pdnn_launch_count": ([], C.c_uint64),
        }
        for name, (args, res) in sig.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = res
        _lib = lib
        return lib


# diagnostics: PDNN_SYNC_CALLS=1 synchronizes the device after every library
# call, so a kernel that never finishes stalls the call that launched it
_SYNC_CALLS = os.environ.get("PDNN_SYNC_CALLS") == "1"


def _check(rc: int, where: str):
    if rc != 0:
        raise PdnnError(rc, where, load_library().pdnn_last_error().decode())
    if _SYNC_CALLS and not torch.cuda.is_current_stream_capturing():
        torch.cuda.synchronize()


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr()


def _dev(t, dtype):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(np.ascontiguousarray(t))
    if t.dtype != dtype:
        raise TypeError(f"expected {dtype}, got {t.dtype}")
    if not t.is_cuda:
        t = t.cuda()
    return t.contiguous()


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def launch_count() -> int:
    return int(load_library().pdnn_launch_count())


# ---------------------------------------------------------------- C-name wrappers
def pdnn_build_csr(n_nodes: int, src: torch.Tensor, dst: torch.Tensor, stream=None):
    """Returns (handle, perm) -- perm[k] = input index of the k-th canonical edge."""
    lib = load_library()
    src, dst = _dev(src, torch.int32), _dev(dst, torch.int32)
    E = int(src.numel())
    perm = torch.empty(E, dtype=torch.int32, device=src.device)
    h = C.c_void_p()
    _check(lib.pdnn_build_csr(int(n_nodes), E, _ptr(src), _ptr(dst), _ptr(perm), _stream(stream), C.byref(h)),
           "pdnn_build_csr")
    return h, perm


def pdnn_graph_free(h):
    if h:
        load_library().pdnn_graph_free(h)


def pdnn_graph_query(h):
    n, m, d, mi, mo = C.c_int32(), C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32()
    _check(load_library().pdnn_graph_query(h, C.byref(n), C.byref(m), C.byref(d), C.byref(mi), C.byref(mo)),
           "pdnn_graph_query")
    return dict(n_nodes=n.value, n_edges=m.value, n_levels=d.value, max_in=mi.value, max_out=mo.value)


def pdnn_workspace_bytes(h, op: int, batch: int = 0) -> int:
    return int(load_library().pdnn_workspace_bytes(h, op, batch))


# ---------------------------------------------------------------- Graph
class Graph:
    """A device graph (pdnn_graph) with its workspace.

    All outputs are torch tensors on the graph's device; inputs may be numpy
    arrays or tensors (host arrays are copied to the device first).
    """

    def __init__(self, n_nodes: int, src, dst, device=None, stream=None):
        self.device = torch.device(device or "cuda")
        with torch.cuda.device(self.device):
            src_t = _dev(src, torch.int32).to(self.device)
            dst_t = _dev(dst, torch.int32).to(self.device)
            self._h, self.perm = pdnn_build_csr(n_nodes, src_t, dst_t, stream)
        q = pdnn_graph_query(self._h)
        self.V, self.E, self.n_levels = q["n_nodes"], q["n_edges"], q["n_levels"]
        self.max_in, self.max_out = q["max_in"], q["max_out"]
        self._ws = None
        self._ws_bytes = 0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                pdnn_graph_free(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def workspace(self, op=PDNN_OP_EVAL_BATCH, batch=0):
        need = pdnn_workspace_bytes(self._h, op, batch)
        if self._ws is None or self._ws_bytes < need:
            self._ws = torch.zeros(need, dtype=torch.uint8, device=self.device)
            self._ws_bytes = need
        return self._ws

    def levels(self, stream=None):
        out = torch.empty(self.V, dtype=torch.int32, device=self.device)
        _check(load_library().pdnn_graph_levels(self._h, _ptr(out), _stream(stream)), "pdnn_graph_levels")
        return out

    def set_costs(self, node_cost, edge_cost, edge_order=PDNN_EDGE_ORDER_INPUT, stream=None):
        c = _dev(node_cost, torch.int64).to(self.device)
        w = _dev(edge_cost, torch.int64).to(self.device)
        _check(load_library().pdnn_graph_set_costs(self._h, _ptr(c), _ptr(w), edge_order, _stream(stream)),
               "pdnn_graph_set_costs")

    def weighted_levels(self, part=None, node_cost=None, edge_cost=None, out=None, stream=None):
        ws = self.workspace()
        p = None if part is None else _dev(part, torch.int32).to(self.device)
        c = None if node_cost is None else _dev(node_cost, torch.int64).to(self.device)
        w = None if edge_cost is None else _dev(edge_cost, torch.int64).to(self.device)
        if out is None:
            out = (torch.empty(self.V, dtype=torch.int64, device=self.device),
                   torch.empty(self.V, dtype=torch.int64, device=self.device))
        tl, bl = out
        _check(load_library().pdnn_weighted_levels(self._h, _ptr(c), _ptr(w), _ptr(p), _ptr(tl), _ptr(bl),
                                                   _ptr(ws), ws.numel(), _stream(stream)),
               "pdnn_weighted_levels")
        return tl, bl

    def critical_path(self, tl, bl, part=None, node_cost=None, edge_cost=None, stream=None):
        ws = self.workspace()
        p = None if part is None else _dev(part, torch.int32).to(self.device)
        c = None if node_cost is None else _dev(node_cost, torch.int64).to(self.device)
        w = None if edge_cost is None else _dev(edge_cost, torch.int64).to(self.device)
        cp = torch.empty(max(self.n_levels, 1), dtype=torch.int32, device=self.device)
        scal = torch.zeros(3, dtype=torch.int64, device=self.device)  # cp_len(i32) | L | hash
        lenp = scal.data_ptr()
        _check(load_library().pdnn_critical_path(self._h, _ptr(c), _ptr(w), _ptr(p), _ptr(tl), _ptr(bl),
                                                 _ptr(cp), lenp, lenp + 8, lenp + 16, _ptr(ws), ws.numel(),
                                                 _stream(stream)),
               "pdnn_critical_path")
        return cp, scal

    @staticmethod
    def unpack_cp(cp, scal):
        """(cp ids as numpy, L, hash) from critical_path's device outputs (syncs)."""
        s = scal.cpu().numpy()
        n = int(s[0] & 0xFFFFFFFF)
        return cp[:n].cpu().numpy(), int(s[1]), int(s[2]) & 0xFFFFFFFFFFFFFFFF

    def slice(self, K: int, node_cost=None, edge_cost=None, stream=None):
        ws = self.workspace()
        c = None if node_cost is None else _dev(node_cost, torch.int64).to(self.device)
        w = None if edge_cost is None else _dev(edge_cost, torch.int64).to(self.device)
        cap = max(self.n_levels, 1)
        cps = torch.empty((K, cap), dtype=torch.int32, device=self.device)
        lens = torch.empty(K, dtype=torch.int32, device=self.device)
        Ls = torch.empty(K, dtype=torch.int64, device=self.device)
        hs = torch.empty(K, dtype=torch.int64, device=self.device)
        _check(load_library().pdnn_slice(self._h, _ptr(c), _ptr(w), int(K), cap, _ptr(cps), _ptr(lens), _ptr(Ls),
                                         _ptr(hs), _ptr(ws), ws.numel(), _stream(stream)),
               "pdnn_slice")
        return cps, lens, Ls, hs

    def memory_potential(self, part, n_pe: int, mem, kind, st, cap_eff, want_mcons=False, stream=None):
        ws = self.workspace()
        p = _dev(part, torch.int32).to(self.device)
        m = _dev(mem, torch.int64).to(self.device)
        k = _dev(kind, torch.uint8).to(self.device)
        s = None if st is None else _dev(st, torch.int64).to(self.device)   # None: st = tl (bound costs)
        cap = _dev(cap_eff, torch.int64).to(self.device)
        P = int(n_pe)
        mpot = torch.empty(self.V, dtype=torch.int64, device=self.device)
        peak = torch.empty(P, dtype=torch.int64, device=self.device)
        ppos = torch.empty(P, dtype=torch.int32, device=self.device)
        fo = torch.empty(P, dtype=torch.int32, device=self.device)
        ob = torch.empty(P, dtype=torch.int64, device=self.device)
        mcons = torch.empty((P, self.V), dtype=torch.int64, device=self.device) if want_mcons else None
        _check(load_library().pdnn_memory_potential(
            self._h, _ptr(p), P, _ptr(m), _ptr(k), _ptr(s), _ptr(cap), _ptr(mpot), _ptr(peak), _ptr(ppos),
            _ptr(fo), _ptr(ob), _ptr(mcons), _ptr(ws), ws.numel(), _stream(stream)),
            "pdnn_memory_potential")
        return dict(mpot=mpot, peak=peak, peak_pos=ppos, first_over=fo, over_bytes=ob, mcons=mcons)

    def slice_clusters(self, K: int, node_cost=None, edge_cost=None, stream=None):
        """Whole of Alg. 1: (cluster_of, members, cl_off, n_clusters) device tensors."""
        ws = self.workspace()
        c = None if node_cost is None else _dev(node_cost, torch.int64).to(self.device)
        w = None if edge_cost is None else _dev(edge_cost, torch.int64).to(self.device)
        cof = torch.empty(self.V, dtype=torch.int32, device=self.device)
        mem = torch.empty(max(self.V, 1), dtype=torch.int32, device=self.device)
        off = torch.empty(self.V + int(K) + 1, dtype=torch.int32, device=self.device)
        nc = torch.zeros(1, dtype=torch.int32, device=self.device)
        _check(load_library().pdnn_slice_clusters(self._h, _ptr(c), _ptr(w), int(K), _ptr(cof), _ptr(mem), _ptr(off),
                                                  _ptr(nc), _ptr(ws), ws.numel(), _stream(stream)),
               "pdnn_slice_clusters")
        return cof, mem, off, nc

    def criticality(self, cluster_of, n_clusters: int, node_cost=None, edge_cost=None, stream=None):
        ws = self.workspace()
        cof = _dev(cluster_of, torch.int32).to(self.device)
        c = None if node_cost is None else _dev(node_cost, torch.int64).to(self.device)
        w = None if edge_cost is None else _dev(edge_cost, torch.int64).to(self.device)
        crit = torch.empty(max(int(n_clusters), 1), dtype=torch.int64, device=self.device)
        _check(load_library().pdnn_criticality(self._h, _ptr(c), _ptr(w), _ptr(cof), int(n_clusters), _ptr(crit),
                                               _ptr(ws), ws.numel(), _stream(stream)),
               "pdnn_criticality")
        return crit[: int(n_clusters)]

    def lflam(self, cluster_of, members, cl_off, n_clusters: int, K: int, node_cost=None, edge_cost=None,
              stream=None):
        """The LFLAM mapping (reading R21).  Returns (part device int32[V],
        log device int32[n_log][3])."""
        ws = self.workspace(PDNN_OP_LFLAM, 0)
        cof = _dev(cluster_of, torch.int32).to(self.device)
        mem = _dev(members, torch.int32).to(self.device)
        off = _dev(cl_off, torch.int32).to(self.device)
        c = None if node_cost is None else _dev(node_cost, torch.int64).to(self.device)
        w = None if edge_cost is None else _dev(edge_cost, torch.int64).to(self.device)
        nc = int(n_clusters)
        part = torch.empty(max(self.V, 1), dtype=torch.int32, device=self.device)
        log = torch.empty((max(nc - int(K), 1), 3), dtype=torch.int32, device=self.device)
        nl = torch.zeros(1, dtype=torch.int32, device=self.device)
        _check(load_library().pdnn_lflam(self._h, _ptr(c), _ptr(w), _ptr(cof), _ptr(mem), _ptr(off), nc, int(K),
                                         _ptr(part), _ptr(log), _ptr(nl), _ptr(ws), ws.numel(), _stream(stream)),
               "pdnn_lflam")
        return part[: self.V], log[: int(nl.item())]

    def refine(self, cluster_of, members, cl_off, n_clusters: int, K: int, part, passes=None, window: int = 64,
               node_cost=None, edge_cost=None, stream=None):
        """The refinement (reading R22): cluster swaps, then `passes` (default K)
        node-level passes.  Returns (part device int32[V], log int64[n][4]
        numpy: (0, A, B, gain) / (1, node, to, L), L of the final placement)."""
        ws = self.workspace(PDNN_OP_REFINE, 0)
        cof = _dev(cluster_of, torch.int32).to(self.device)
        mem = _dev(members, torch.int32).to(self.device)
        off = _dev(cl_off, torch.int32).to(self.device)
        p = _dev(part, torch.int32).to(self.device).clone()
        c = None if node_cost is None else _dev(node_cost, torch.int64).to(self.device)
        w = None if edge_cost is None else _dev(edge_cost, torch.int64).to(self.device)
        ps = int(K) if passes is None else int(passes)
        cap = int(n_clusters) + 2 * (self.n_levels + 1) * ps + 16
        log = np.zeros((cap, 4), np.int64)
        nl, L = C.c_int32(), C.c_int64()
        _check(load_library().pdnn_refine(self._h, _ptr(c), _ptr(w), _ptr(cof), _ptr(mem), _ptr(off), int(n_clusters),
                                          int(K), ps, int(window), _ptr(p), log.ctypes.data, cap, C.byref(nl),
                                          C.byref(L), _ptr(ws), ws.numel(), _stream(stream)), "pdnn_refine")
        assert nl.value <= cap
        return p[: self.V], log[: nl.value].copy(), L.value

    def resolve_overflow(self, part, n_pe: int, mem, kind, cap_eff, max_moves=None, node_cost=None, edge_cost=None,
                         stream=None):
        """The overflow handler (reading R20).  Returns (final part (device int32),
        moves int32[n][3] numpy, resolved bool)."""
        ws = self.workspace(PDNN_OP_RESOLVE_OVERFLOW, 0)
        p = _dev(part, torch.int32).to(self.device).clone()
        m = _dev(mem, torch.int64).to(self.device)
        k = _dev(kind, torch.uint8).to(self.device)
        cap = np.ascontiguousarray(np.asarray(cap_eff, dtype=np.int64))
        c = None if node_cost is None else _dev(node_cost, torch.int64).to(self.device)
        w = None if edge_cost is None else _dev(edge_cost, torch.int64).to(self.device)
        mm = self.V if max_moves is None else int(max_moves)
        moves = np.zeros((max(mm, 1), 3), np.int32)
        nm, res = C.c_int32(), C.c_int32()
        _check(load_library().pdnn_resolve_overflow(
            self._h, _ptr(c), _ptr(w), _ptr(m), _ptr(k), int(n_pe), cap.ctypes.data, _ptr(p), mm,
            moves.ctypes.data, C.byref(nm), C.byref(res), _ptr(ws), ws.numel(), _stream(stream)),
            "pdnn_resolve_overflow")
        return p, moves[: nm.value].copy(), bool(res.value)

    def validate(self, node_cost=None, edge_cost=None, part=None, n_pe=0, mem=None, kind=None, st=None,
                 stream=None):
        """pdnn_validate: raises PdnnError on a violated data precondition."""
        def d(x, dt):
            return None if x is None else _dev(x, dt).to(self.device)
        # keep every converted tensor referenced until the (synchronous) call returns
        args = [d(node_cost, torch.int64), d(edge_cost, torch.int64), d(part, torch.int32)]
        more = [d(mem, torch.int64), d(kind, torch.uint8), d(st, torch.int64)]
        _check(load_library().pdnn_validate(self._h, *[_ptr(x) for x in args], int(n_pe), *[_ptr(x) for x in more],
                                            _stream(stream)), "pdnn_validate")

    def emulate(self, part, n_pe: int, node_cost=None, edge_cost=None, stream=None):
        """The TF FIFO scheduler emulator: (st, ft, makespan) device tensors."""
        ws = self.workspace()
        need = pdnn_workspace_bytes(self._h, PDNN_OP_EMULATE, 0)
        if ws.numel() < need:
            ws = self.workspace(PDNN_OP_EMULATE, 0)
        p = _dev(part, torch.int32).to(self.device)
        c = None if node_cost is None else _dev(node_cost, torch.int64).to(self.device)
        w = None if edge_cost is None else _dev(edge_cost, torch.int64).to(self.device)
        st = torch.empty(self.V, dtype=torch.int64, device=self.device)
        ft = torch.empty(self.V, dtype=torch.int64, device=self.device)
        mk = torch.zeros(1, dtype=torch.int64, device=self.device)
        _check(load_library().pdnn_emulate(self._h, _ptr(c), _ptr(w), _ptr(p), int(n_pe), _ptr(st), _ptr(ft),
                                           _ptr(mk), _ptr(ws), ws.numel(), _stream(stream)),
               "pdnn_emulate")
        return st, ft, mk

    def eval_batch(self, parts, n_pe: int, mem, kind, cap_eff, node_cost=None, edge_cost=None, out=None,
                   stream=None, schedule=PDNN_SCHEDULE_LEVEL):
        """parts: uint8 [B][V] (device or host).  Returns a uint8 device tensor
        of B * 432 bytes (view on host with EVAL_RESULT_DTYPE)."""
        pt = _dev(parts, torch.uint8).to(self.device)
        B = int(pt.shape[0]) if pt.dim() == 2 else 0
        ws = self.workspace(PDNN_OP_EVAL_BATCH_EMULATED if schedule else PDNN_OP_EVAL_BATCH, B)
        m = _dev(mem, torch.int64).to(self.device)
        k = _dev(kind, torch.uint8).to(self.device)
        cap = _dev(cap_eff, torch.int64).to(self.device)
        c = None if node_cost is None else _dev(node_cost, torch.int64).to(self.device)
        w = None if edge_cost is None else _dev(edge_cost, torch.int64).to(self.device)
        if out is None:
            out = torch.zeros(B * EVAL_RESULT_DTYPE.itemsize, dtype=torch.uint8, device=self.device)
        _check(load_library().pdnn_eval_batch(self._h, _ptr(c), _ptr(w), _ptr(m), _ptr(k), int(n_pe), _ptr(cap), B,
                                              _ptr(pt), _ptr(out), int(schedule), _ptr(ws), ws.numel(),
                                              _stream(stream)),
               "pdnn_eval_batch")
        return out

    @staticmethod
    def results_to_numpy(out: torch.Tensor) -> np.ndarray:
        return out.cpu().numpy().view(EVAL_RESULT_DTYPE)
