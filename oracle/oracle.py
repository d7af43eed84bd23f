"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper of ``oracle/oracle.c``.

Argument marshalling only; every computation happens in the C oracle, whose
functions cite the PAPER.md passages they transcribe.  Edge costs are passed in
the caller's input edge order (the order of ``src``/``dst`` given to the
constructor).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

REMOVED = -1
UNASSIGNED = -2
KIND_NORMAL, KIND_RESIDUAL, KIND_REFERENCE = 0, 1, 2
MAX_PE = 16

_ERR = {0: "OK", -1: "EINVAL", -2: "ECYCLE", -3: "ENOMEM", -5: "EOVERFLOW"}

EVAL_DTYPE = np.dtype(
    [
        ("L", "<i8"),
        ("cut_comm", "<i8"),
        ("cp_hash", "<u8"),
        ("cp_len", "<i4"),
        ("cp_start", "<i4"),
        ("cp_end", "<i4"),
        ("overflow_mask", "<i4"),
        ("peak", "<i8", (MAX_PE,)),
        ("over_bytes", "<i8", (MAX_PE,)),
        ("peak_pos", "<i4", (MAX_PE,)),
        ("first_over_pos", "<i4", (MAX_PE,)),
        ("makespan", "<i8"),
    ]
)


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"oracle {where}: {_ERR.get(code, code)}")
        self.code = code
        self.name = _ERR.get(code, str(code))


def build_lib(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain C11, -O2, pthreads)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-pthread", "-o", tmp, _SRC]
        )
        os.replace(tmp, _LIB)
    return _LIB


_lib = None
_lock = threading.Lock()


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = C.CDLL(build_lib())
            P = C.c_void_p
            lib.or_build.argtypes = [C.c_int32, C.c_int64, P, P, C.POINTER(P)]
            lib.or_free.argtypes = [P]
            lib.or_free.restype = None
            lib.or_n_levels.argtypes = [P]
            lib.or_n_levels.restype = C.c_int32
            lib.or_levels.argtypes = [P, P]
            lib.or_levels.restype = None
            lib.or_topo.argtypes = [P, P]
            lib.or_topo.restype = None
            lib.or_weighted_levels.argtypes = [P, P, P, P, P, P]
            lib.or_critical_path.argtypes = [P] * 6 + [P, P, P, P]
            lib.or_slice.argtypes = [P, P, P, C.c_int32, C.c_int32, P, P, P, P]
            lib.or_memory.argtypes = [P, P, C.c_int32] + [P] * 11
            lib.or_eval_batch.argtypes = [P, P, P, P, P, C.c_int32, P, C.c_int32, P, P, C.c_int32, C.c_int32]
            lib.or_emulate.argtypes = [P, P, P, P, C.c_int32, P, P, P, P]
            lib.or_slice_clusters.argtypes = [P, P, P, C.c_int32, P, P, P, P]
            lib.or_criticality.argtypes = [P, P, P, P, C.c_int32, P]
            lib.or_lflam.argtypes = [P, P, P, P, P, P, C.c_int32, C.c_int32, P, P, P]
            lib.or_refine.argtypes = [P] * 6 + [C.c_int32] * 4 + [P, P, C.c_int32, P, P]
            lib.or_mpot_at.argtypes = [P, P, P, P, P, C.c_int32, C.c_int32, P]
            lib.or_resolve_overflow.argtypes = [P, P, P, P, P, C.c_int32, P, P, C.c_int32, P, P, P]
            _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


class OracleGraph:
    """A DAG built by the oracle (Kahn levels, validation)."""

    def __init__(self, n_nodes: int, src, dst):
        lib = _load()
        self.src = _i32(src)
        self.dst = _i32(dst)
        self.V = int(n_nodes)
        self.E = int(self.src.shape[0])
        h = C.c_void_p()
        rc = lib.or_build(self.V, self.E, _p(self.src), _p(self.dst), C.byref(h))
        if rc:
            raise OracleError(rc, "build")
        self._h = h
        self.n_levels = int(lib.or_n_levels(h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.or_free(h)
            self._h = None

    def levels(self) -> np.ndarray:
        out = np.empty(self.V, np.int32)
        _load().or_levels(self._h, _p(out))
        return out

    def topo(self) -> np.ndarray:
        out = np.empty(self.V, np.int32)
        _load().or_topo(self._h, _p(out))
        return out

    def weighted_levels(self, c, w, part=None):
        c, w = _i64(c), _i64(w)
        part = None if part is None else _i32(part)
        tl = np.empty(self.V, np.int64)
        bl = np.empty(self.V, np.int64)
        rc = _load().or_weighted_levels(self._h, _p(c), _p(w), _p(part), _p(tl), _p(bl))
        if rc:
            raise OracleError(rc, "weighted_levels")
        return tl, bl

    def critical_path(self, c, w, part, tl, bl):
        c, w, tl, bl = _i64(c), _i64(w), _i64(tl), _i64(bl)
        part = None if part is None else _i32(part)
        cp = np.empty(max(self.n_levels, 1), np.int32)
        n = C.c_int32()
        L = C.c_int64()
        h = C.c_uint64()
        rc = _load().or_critical_path(
            self._h, _p(c), _p(w), _p(part), _p(tl), _p(bl), _p(cp), C.byref(n), C.byref(L), C.byref(h)
        )
        if rc:
            raise OracleError(rc, "critical_path")
        return cp[: n.value].copy(), int(L.value), int(h.value)

    def slice(self, c, w, K: int):
        c, w = _i64(c), _i64(w)
        cap = max(self.n_levels, 1)
        cps = np.empty((K, cap), np.int32)
        lens = np.empty(K, np.int32)
        Ls = np.empty(K, np.int64)
        hs = np.empty(K, np.uint64)
        rc = _load().or_slice(self._h, _p(c), _p(w), int(K), cap, _p(cps), _p(lens), _p(Ls), _p(hs))
        if rc:
            raise OracleError(rc, "slice")
        return [cps[j, : lens[j]].copy() for j in range(K)], Ls, hs

    def memory(self, part, n_pe: int, mem, kind, st, cap_eff, want_mcons=False):
        part, mem, st, cap_eff = _i32(part), _i64(mem), _i64(st), _i64(cap_eff)
        kind = np.ascontiguousarray(kind, dtype=np.uint8)
        P = int(n_pe)
        mpot = np.empty(self.V, np.int64)
        peak = np.empty(P, np.int64)
        ppos = np.empty(P, np.int32)
        fo = np.empty(P, np.int32)
        ob = np.empty(P, np.int64)
        order = np.empty(self.V, np.int32)
        mcons = np.empty((P, self.V), np.int64) if want_mcons else None
        rc = _load().or_memory(
            self._h, _p(part), P, _p(mem), _p(kind), _p(st), _p(cap_eff),
            _p(mpot), _p(peak), _p(ppos), _p(fo), _p(ob), _p(mcons), _p(order),
        )
        if rc:
            raise OracleError(rc, "memory")
        return dict(mpot=mpot, peak=peak, peak_pos=ppos, first_over=fo, over_bytes=ob,
                    mcons=mcons, order=order)

    def slice_clusters(self, c, w, K: int):
        """Whole of Alg. 1 (reading R18): (cluster_of, list of clusters as node-id
        arrays in path order; the first K are the primaries)."""
        c, w = _i64(c), _i64(w)
        cof = np.empty(self.V, np.int32)
        mem = np.empty(max(self.V, 1), np.int32)
        off = np.empty(self.V + K + 2, np.int32)
        nc = C.c_int32()
        rc = _load().or_slice_clusters(self._h, _p(c), _p(w), int(K), _p(cof), _p(mem), _p(off), C.byref(nc))
        if rc:
            raise OracleError(rc, "slice_clusters")
        k = nc.value
        return cof, [mem[off[i]:off[i + 1]].copy() for i in range(k)]

    def criticality(self, c, w, cluster_of, n_clusters: int):
        c, w, cof = _i64(c), _i64(w), _i32(cluster_of)
        crit = np.empty(max(n_clusters, 1), np.int64)
        rc = _load().or_criticality(self._h, _p(c), _p(w), _p(cof), int(n_clusters), _p(crit))
        if rc:
            raise OracleError(rc, "criticality")
        return crit[:n_clusters]

    def lflam(self, c, w, cluster_of, clusters, K: int):
        """LFLAM mapping (Alg. 2, reading R21): (part, log [(cluster, phase, pe)])."""
        c, w, cof = _i64(c), _i64(w), _i32(cluster_of)
        members = np.concatenate(clusters).astype(np.int32) if len(clusters) else np.zeros(0, np.int32)
        off = np.zeros(len(clusters) + 1, np.int32)
        off[1:] = np.cumsum([len(x) for x in clusters])
        part = np.empty(self.V, np.int32)
        log = np.zeros((max(len(clusters), 1), 3), np.int32)
        nl = C.c_int32()
        rc = _load().or_lflam(self._h, _p(c), _p(w), _p(cof), _p(members), _p(off), len(clusters), int(K), _p(part),
                              _p(log), C.byref(nl))
        if rc:
            raise OracleError(rc, "lflam")
        return part, log[: nl.value].copy()

    def refine(self, c, w, cluster_of, clusters, K: int, part, passes=None, window: int = 64):
        """Refinement (appendix "Complexity of Refinement", reading R22): cluster
        swaps, then `passes` (default K) node-level passes.  Returns (part, log
        int64 [n][4]: (0, A, B, gain) / (1, node, to, L), L of the final part)."""
        c, w, cof = _i64(c), _i64(w), _i32(cluster_of)
        members = np.concatenate(clusters).astype(np.int32) if len(clusters) else np.zeros(0, np.int32)
        off = np.zeros(len(clusters) + 1, np.int32)
        off[1:] = np.cumsum([len(x) for x in clusters])
        part = np.array(part, dtype=np.int32, copy=True)
        cap = len(clusters) + 4 * (self.n_levels + 1) * (K if passes is None else passes) + 16
        log = np.zeros((cap, 4), np.int64)
        nl = C.c_int32()
        L = C.c_int64()
        rc = _load().or_refine(self._h, _p(c), _p(w), _p(cof), _p(members), _p(off), len(clusters), int(K),
                               int(K if passes is None else passes), int(window), _p(part), _p(log), cap,
                               C.byref(nl), C.byref(L))
        if rc:
            raise OracleError(rc, "refine")
        assert nl.value <= cap
        return part, log[: nl.value].copy(), L.value

    def mpot_at(self, part, mem, kind, pos, q: int, i: int):
        """M_pot(n, t) of every node at visit position i on PE q (reading R20)."""
        part, mem, pos = _i32(part), _i64(mem), _i32(pos)
        kind = np.ascontiguousarray(kind, dtype=np.uint8)
        a = np.empty(self.V, np.int64)
        _load().or_mpot_at(self._h, _p(part), _p(mem), _p(kind), _p(pos), int(q), int(i), _p(a))
        return a

    def resolve_overflow(self, c, w, mem, kind, n_pe, cap_eff, part, max_moves=None):
        """The overflow handler (reading R20): (final part, moves [(node, from, to)]
        with to = -1 for rejected candidates, resolved)."""
        c, w, mem, cap_eff = _i64(c), _i64(w), _i64(mem), _i64(cap_eff)
        kind = np.ascontiguousarray(kind, dtype=np.uint8)
        part = np.array(part, dtype=np.int32, copy=True)
        mm = self.V if max_moves is None else int(max_moves)
        moves = np.zeros((max(mm, 1), 3), np.int32)
        nm, res = C.c_int32(), C.c_int32()
        rc = _load().or_resolve_overflow(self._h, _p(c), _p(w), _p(mem), _p(kind), int(n_pe), _p(cap_eff), _p(part),
                                         mm, _p(moves), C.byref(nm), C.byref(res))
        if rc:
            raise OracleError(rc, "resolve_overflow")
        return part, moves[: nm.value].copy(), bool(res.value)

    def emulate(self, c, w, part, n_pe):
        """The TF FIFO scheduler emulator (reading R17):
        returns st, ft (int64 [V]), the makespan and the largest ready queue."""
        c, w, part = _i64(c), _i64(w), _i32(part)
        st = np.empty(self.V, np.int64)
        ft = np.empty(self.V, np.int64)
        mk = C.c_int64()
        mq = C.c_int32()
        rc = _load().or_emulate(self._h, _p(c), _p(w), _p(part), int(n_pe), _p(st), _p(ft), C.byref(mk), C.byref(mq))
        if rc:
            raise OracleError(rc, "emulate")
        return st, ft, int(mk.value), int(mq.value)

    def eval_batch(self, c, w, mem, kind, n_pe, cap_eff, parts, n_threads=None, schedule=0):
        c, w, mem, cap_eff = _i64(c), _i64(w), _i64(mem), _i64(cap_eff)
        kind = np.ascontiguousarray(kind, dtype=np.uint8)
        parts = np.ascontiguousarray(parts, dtype=np.uint8)
        B = int(parts.shape[0])
        out = np.zeros(B, EVAL_DTYPE)
        if n_threads is None:
            n_threads = len(os.sched_getaffinity(0))
        rc = _load().or_eval_batch(
            self._h, _p(c), _p(w), _p(mem), _p(kind), int(n_pe), _p(cap_eff), B, _p(parts),
            _p(out), int(n_threads), int(schedule),
        )
        if rc:
            raise OracleError(rc, "eval_batch")
        return out
