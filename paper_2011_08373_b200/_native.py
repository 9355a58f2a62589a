"""ctypes binding of libgrsolve.so (include/gr.h) -- argument marshalling only.

Every step of the Solve path runs in the CUDA kernels behind the C-ABI; this
module turns torch device tensors into the plain pointers gr.h declares and
passes torch's current stream.  There is no CPU fallback: if the library is
missing or no CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GRSOLVE_LIB") or os.path.join(HERE, "libgrsolve.so")  # override: dev A/B builds

GR_OK, GR_EINVAL, GR_ETOOBIG, GR_ECUDA, GR_ENOMEM, GR_EWORKSPACE = 0, -1, -2, -3, -4, -5
GR_SAT, GR_UNSAT, GR_SAT_NEG_VIOLATED, GR_BADINPUT, GR_UNSUPPORTED = 0, 1, 2, 3, 4
GR_FLAG_EXHAUSTIVE = 1
GR_FLAG_WEIGHTED_GREEDY = 2
GR_FLAG_NO_PRUNE = 4
PMS, MHS, GREEDY = 0, 1, 2

EXPORTED = [
    "gr_workspace_bytes", "gr_solve_pms", "gr_mhs_exact", "gr_mhs_greedy", "gr_exact_prepare",
    "gr_exact_level", "gr_exact_level_keys", "gr_exact_finish", "gr_bitmatrix_ld",
    "gr_pack_varmajor", "gr_pack_clausemajor", "gr_greedy_matrix_workspace_bytes",
    "gr_mhs_greedy_matrix", "gr_greedy_count_shard", "gr_last_error", "gr_version",
    "gr_profile", "gr_profile_read", "gr_launch_count", "gr_solve", "gr_solve_pms_mhs",
    "gr_greedy_shard_workspace_bytes", "gr_greedy_shard_begin", "gr_greedy_shard_step",
    "gr_greedy_shard_state", "gr_greedy_shard_private", "gr_greedy_shard_remove",
    "gr_greedy_shard_finalize", "gr_pair_prepare", "gr_pair_level", "gr_pair_level_keys",
    "gr_pair_finish", "gr_greedy_lists_workspace_bytes", "gr_mhs_greedy_lists",
]
GR_STRATEGY_MHS, GR_STRATEGY_MAXSAT, GR_STRATEGY_MHS_FINAL = 0, 1, 2


class GrBatch(C.Structure):
    _fields_ = [
        ("B", C.c_int32), ("W", C.c_int32), ("total_clauses", C.c_int64),
        ("max_clauses", C.c_int32), ("flags", C.c_uint32),
        ("m", C.c_void_p), ("off", C.c_void_p), ("n_pos", C.c_void_p), ("masks", C.c_void_p),
        ("w", C.c_void_p), ("wstride", C.c_int32), ("k_start", C.c_void_p),
    ]


class GrResult(C.Structure):
    _fields_ = [("assign", C.c_void_p), ("cost", C.c_void_p), ("status", C.c_void_p),
                ("decided", C.c_void_p)]


class GrKernelStat(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("launches", C.c_int64), ("ms", C.c_double),
                ("work", C.c_uint64 * 8)]


class GrBitmatrix(C.Structure):
    _fields_ = [("m", C.c_int32), ("n_pos", C.c_int64), ("ld", C.c_int64), ("bits", C.c_void_p),
                ("n_neg", C.c_int32), ("neg", C.c_void_p), ("pos_off", C.c_void_p),
                ("pos_var", C.c_void_p), ("var_bytes", C.c_int32), ("w", C.c_void_p)]


_lib = None


def lib():
    """Load libgrsolve.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t
        L.gr_workspace_bytes.argtypes = [vp, C.c_int]
        L.gr_workspace_bytes.restype = sz
        for f in (L.gr_solve_pms, L.gr_mhs_exact, L.gr_mhs_greedy):
            f.argtypes = [vp, vp, vp, sz, vp]
            f.restype = C.c_int
        L.gr_exact_prepare.argtypes = [vp, C.c_int, vp, vp, sz, vp, vp]
        L.gr_solve.argtypes = [vp, C.c_int, vp, vp, vp, sz, vp]
        L.gr_solve_pms_mhs.argtypes = [vp, vp, vp, vp, sz, vp, vp]
        L.gr_solve_pms_mhs.restype = C.c_int
        L.gr_solve.restype = C.c_int
        L.gr_profile.argtypes = [C.c_int]
        L.gr_profile.restype = C.c_int
        L.gr_profile_read.argtypes = [vp, C.c_int]
        L.gr_profile_read.restype = C.c_int
        L.gr_launch_count.restype = C.c_ulonglong
        L.gr_exact_level.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, sz, vp]
        L.gr_exact_level_keys.argtypes = [vp, C.c_int, vp]
        L.gr_exact_level_keys.restype = vp
        L.gr_exact_finish.argtypes = [vp, C.c_int, C.c_int, vp, vp, sz, vp, vp]
        L.gr_bitmatrix_ld.argtypes = [i64]
        L.gr_bitmatrix_ld.restype = i64
        L.gr_pack_varmajor.argtypes = [i32, i64, vp, vp, C.c_int, vp, i64, vp, vp]
        L.gr_pack_clausemajor.argtypes = [i32, i64, vp, vp, C.c_int, vp, vp, vp]
        L.gr_greedy_matrix_workspace_bytes.argtypes = [vp]
        L.gr_greedy_matrix_workspace_bytes.restype = sz
        L.gr_mhs_greedy_matrix.argtypes = [vp, vp, vp, vp, vp, vp, sz, vp]
        L.gr_greedy_count_shard.argtypes = [vp, vp, vp, vp]
        L.gr_greedy_shard_workspace_bytes.argtypes = [vp]
        L.gr_greedy_shard_workspace_bytes.restype = sz
        L.gr_greedy_shard_begin.argtypes = [vp, vp, vp, sz, vp]
        L.gr_greedy_shard_step.argtypes = [vp, vp, vp, sz, vp]
        L.gr_greedy_shard_state.argtypes = [vp, vp, sz, vp, vp, vp, vp]
        L.gr_greedy_shard_private.argtypes = [vp, i32, vp, vp, sz, vp]
        L.gr_greedy_shard_remove.argtypes = [vp, i32, vp, sz, vp]
        L.gr_greedy_shard_finalize.argtypes = [vp, vp, vp, vp, vp, sz, vp]
        for f in (L.gr_greedy_shard_begin, L.gr_greedy_shard_step, L.gr_greedy_shard_state,
                  L.gr_greedy_shard_private, L.gr_greedy_shard_remove, L.gr_greedy_shard_finalize):
            f.restype = C.c_int
        if hasattr(L, "gr_pair_prepare"):
            L.gr_pair_prepare.argtypes = [vp, vp, vp, vp, sz, vp, vp]
            L.gr_pair_level.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, sz, vp]
            L.gr_pair_level_keys.argtypes = [vp, vp, C.c_int]
            L.gr_pair_level_keys.restype = vp
            L.gr_pair_finish.argtypes = [vp, C.c_int, vp, vp, vp, sz, vp, vp]
            for f in (L.gr_pair_prepare, L.gr_pair_level, L.gr_pair_finish):
                f.restype = C.c_int
        if hasattr(L, "gr_mhs_greedy_lists"):  # (older A/B builds via GRSOLVE_LIB lack it)
            L.gr_greedy_lists_workspace_bytes.argtypes = [vp]
            L.gr_greedy_lists_workspace_bytes.restype = sz
            L.gr_mhs_greedy_lists.argtypes = [vp, vp, vp, vp, vp, vp, sz, vp]
            L.gr_mhs_greedy_lists.restype = C.c_int
        L.gr_last_error.restype = C.c_char_p
        L.gr_version.restype = C.c_char_p
        for f in (L.gr_exact_prepare, L.gr_exact_level, L.gr_exact_finish, L.gr_pack_varmajor,
                  L.gr_pack_clausemajor, L.gr_mhs_greedy_matrix, L.gr_greedy_count_shard):
            f.restype = C.c_int
        _lib = L
    return _lib


class GrError(RuntimeError):
    pass


def _check(rc: int, what: str):
    if rc != GR_OK:
        raise GrError(f"{what} failed ({rc}): {lib().gr_last_error().decode()}")


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise GrError("libgrsolve needs a CUDA device (there is no CPU fallback)")
    return torch


def _ptr(t) -> Optional[int]:
    return None if t is None else int(t.data_ptr())


def _stream(stream=None) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


# ---------------------------------------------------------------------------
# batches
# ---------------------------------------------------------------------------
@dataclass
class DeviceBatch:
    """A synth.ClauseBatch resident in device memory (torch tensors)."""

    m: "object"
    off: "object"
    n_pos: "object"
    masks: "object"
    w: "object"
    B: int
    W: int
    total_clauses: int
    max_clauses: int
    wstride: int = 0
    flags: int = 0
    k_start: "object" = None  # optional int32 [B] start levels (incremental Solve, f2)

    @staticmethod
    def from_host(cb, device="cuda", flags: int = 0, weighted: bool = True,
                  non_blocking: bool = False, pinned: bool = False) -> "DeviceBatch":
        torch = _torch()

        def dev(a, dt):
            t = torch.from_numpy(np.ascontiguousarray(a).view(dt))
            if pinned:
                t = t.pin_memory()
            return t.to(device, non_blocking=non_blocking)

        n = np.diff(cb.off)
        w = None
        ws = 0
        if weighted and cb.w is not None:
            w = dev(cb.w.astype(np.uint32).view(np.int32), np.int32)
            ws = int(cb.w.shape[1])
        masks = cb.masks if cb.masks.shape[0] else np.zeros((1, cb.W), np.uint64)
        return DeviceBatch(
            m=dev(cb.m.astype(np.int32), np.int32), off=dev(cb.off.astype(np.int64), np.int64),
            n_pos=dev(cb.n_pos.astype(np.int32), np.int32),
            masks=dev(masks.astype(np.uint64).view(np.int64), np.int64), w=w, B=cb.B, W=cb.W,
            total_clauses=int(cb.off[-1]), max_clauses=int(n.max()) if n.size else 0,
            wstride=ws, flags=flags)

    def struct(self, weighted: bool = True) -> GrBatch:
        return GrBatch(self.B, self.W, self.total_clauses, self.max_clauses, self.flags,
                       _ptr(self.m), _ptr(self.off), _ptr(self.n_pos), _ptr(self.masks),
                       _ptr(self.w) if weighted else None, self.wstride if weighted else 0,
                       _ptr(self.k_start))


@dataclass
class DeviceResult:
    assign: "object"  # int64 view of uint64 [B, W]
    cost: "object"
    status: "object"
    decided: "object"

    @staticmethod
    def empty(B: int, W: int, device="cuda") -> "DeviceResult":
        torch = _torch()
        return DeviceResult(
            torch.zeros((B, W), dtype=torch.int64, device=device),
            torch.zeros(B, dtype=torch.int64, device=device),
            torch.zeros(B, dtype=torch.int32, device=device),
            torch.zeros(B, dtype=torch.int64, device=device))

    def struct(self) -> GrResult:
        return GrResult(_ptr(self.assign), _ptr(self.cost), _ptr(self.status), _ptr(self.decided))

    def to_host(self, stream=None):
        """-> dict of numpy arrays (assign/cost/decided as uint64).  ``stream``:
        the stream the result was produced on (default: the current stream of
        its device)."""
        return to_host_many([self], stream)[0]


def to_host_many(results, stream=None):
    """Several DeviceResults -> dicts of numpy arrays with one synchronisation
    per device: every field is copied (non-blocking) into pinned host memory
    on the stream that produced it -- ``stream`` if given (a torch stream, for
    results of calls made with stream=...), else the current stream of the
    result's device -- then each of those streams is synchronised once."""
    torch = _torch()
    pend, used = [], {}
    for r in results:
        dev = r.status.device
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        used[(dev, id(st))] = st
        d = {}
        with torch.cuda.stream(st):
            for k in ("assign", "cost", "status", "decided"):
                t = getattr(r, k)
                h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                h.copy_(t, non_blocking=True)
                d[k] = h
        pend.append(d)
    for st in used.values():
        st.synchronize()
    out = []
    for d in pend:
        out.append({"assign": d["assign"].numpy().view(np.uint64),
                    "cost": d["cost"].numpy().view(np.uint64),
                    "status": d["status"].numpy(),
                    "decided": d["decided"].numpy().view(np.uint64)})
    return out


_ws_cache = {}


def workspace(nbytes: int, device="cuda", tag: str = "default"):
    """A cached uint8 device buffer of at least nbytes."""
    torch = _torch()
    key = (str(device), tag)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
        _ws_cache[key] = buf
    return buf


def _solve(fn_name: str, which: int, db: DeviceBatch, out: Optional[DeviceResult], stream):
    L = lib()
    weighted = which == PMS
    b = db.struct(weighted)
    nbytes = L.gr_workspace_bytes(C.byref(b), which)
    if nbytes == 0:
        raise GrError("gr_workspace_bytes rejected the batch")
    ws = workspace(nbytes, db.m.device, tag=f"exact{which}")
    if out is None:
        out = DeviceResult.empty(db.B, db.W, db.m.device)
    r = out.struct()
    _check(getattr(L, fn_name)(C.byref(b), C.byref(r), _ptr(ws), ws.numel(), _stream(stream)),
           fn_name)
    return out


def solve_pms(db: DeviceBatch, out: Optional[DeviceResult] = None, stream=None) -> DeviceResult:
    """(a) exact PMS / WPMS (gr_solve_pms)."""
    return _solve("gr_solve_pms", PMS, db, out, stream)


def mhs_exact(db: DeviceBatch, out: Optional[DeviceResult] = None, stream=None) -> DeviceResult:
    """(b) exact MHS of phi+ (gr_mhs_exact)."""
    return _solve("gr_mhs_exact", MHS, db, out, stream)


_side_streams = {}


def solve_pms_mhs(db: DeviceBatch, out_pms: Optional[DeviceResult] = None,
                  out_mhs: Optional[DeviceResult] = None, stream=None):
    """(a) + (b) at once (gr_solve_pms_mhs): PMS on the current stream, MHS on a
    side stream of the same device; the current stream waits for both."""
    torch = _torch()
    L = lib()
    b = db.struct(True)
    nbytes = L.gr_workspace_bytes(C.byref(b), PMS)
    if nbytes == 0:
        raise GrError("gr_workspace_bytes rejected the batch")
    half = (nbytes + 255) // 256 * 256
    ws = workspace(2 * half, db.m.device, tag="pair")
    dev = db.m.device
    out_pms = out_pms if out_pms is not None else DeviceResult.empty(db.B, db.W, dev)
    out_mhs = out_mhs if out_mhs is not None else DeviceResult.empty(db.B, db.W, dev)
    s1 = stream if stream is not None else torch.cuda.current_stream(dev)
    s2 = _side_streams.get(str(dev))
    if s2 is None:
        s2 = _side_streams[str(dev)] = torch.cuda.Stream(device=dev)
    s2.wait_stream(s1)  # inputs produced on the current stream
    r1, r2 = out_pms.struct(), out_mhs.struct()
    _check(L.gr_solve_pms_mhs(C.byref(b), C.byref(r1), C.byref(r2), _ptr(ws), ws.numel(),
                              int(s1.cuda_stream), int(s2.cuda_stream)), "gr_solve_pms_mhs")
    s1.wait_stream(s2)
    return out_pms, out_mhs


def mhs_greedy(db: DeviceBatch, out: Optional[DeviceResult] = None, stream=None) -> DeviceResult:
    """(c) greedy mhs of phi+ (gr_mhs_greedy); weighted when db.flags has
    GR_FLAG_WEIGHTED_GREEDY and db.w is set (f4)."""
    L = lib()
    b = db.struct(True)
    ws = workspace(256, db.m.device, tag="greedy")
    if out is None:
        out = DeviceResult.empty(db.B, db.W, db.m.device)
    r = out.struct()
    _check(L.gr_mhs_greedy(C.byref(b), C.byref(r), _ptr(ws), ws.numel(), _stream(stream)),
           "gr_mhs_greedy")
    return out


_greedy_streams = {}


def solve_step(db: DeviceBatch, out_pms: Optional[DeviceResult] = None,
               out_mhs: Optional[DeviceResult] = None, out_greedy: Optional[DeviceResult] = None,
               stream=None):
    """One Solve step of a batch: exact PMS + MHS (gr_solve_pms_mhs) and the
    greedy mhs (gr_mhs_greedy).  The two are independent, so the greedy is
    launched first on a side stream of the device: its CTAs run beside the
    pack and the start of the exact solve's persistent grid instead of after
    it.  ``stream`` (default: the current stream) waits for both."""
    torch = _torch()
    dev = db.m.device
    s1 = stream if stream is not None else torch.cuda.current_stream(dev)
    g = _greedy_streams.get(str(dev))
    if g is None:
        g = _greedy_streams[str(dev)] = torch.cuda.Stream(device=dev)
    g.wait_stream(s1)  # inputs produced on s1
    out_greedy = mhs_greedy(db, out_greedy, stream=g)
    out_pms, out_mhs = solve_pms_mhs(db, out_pms, out_mhs, stream=s1)
    s1.wait_stream(g)
    return out_pms, out_mhs, out_greedy


class StepGraph:
    """solve_step of one batch captured once as a CUDA graph (launch-bound
    small batches: one replay instead of six launches and two stream forks).
    The graph reads the batch's device buffers and writes ``outs`` in place:
    refill ``db``'s tensors (same shapes) and replay() for the next step.
    The exact solvers' ticket ring is cleared by the pack on every launch, so
    replays never see an earlier run's entries."""

    def __init__(self, db: DeviceBatch, outs=None):
        torch = _torch()
        dev = db.m.device
        self.db = db
        self.outs = list(outs) if outs is not None else [DeviceResult.empty(db.B, db.W, dev) for _ in range(3)]
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):  # warm-up: workspaces, launch attributes
            solve_step(db, *self.outs)
        torch.cuda.current_stream(dev).wait_stream(s)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            solve_step(db, *self.outs)

    def replay(self):
        self.graph.replay()
        return self.outs


def solve(db: DeviceBatch, strategy: int = GR_STRATEGY_MHS, out: Optional[DeviceResult] = None,
          fell_back=None, stream=None) -> DeviceResult:
    """The composite Solve (gr_solve): mhs strategy with MaxSAT fallback, or MaxSAT."""
    torch = _torch()
    L = lib()
    b = db.struct(True)
    nbytes = L.gr_workspace_bytes(C.byref(b), PMS)
    if nbytes == 0:
        raise GrError("gr_workspace_bytes rejected the batch")
    ws = workspace(nbytes, db.m.device, tag="exact0")
    if out is None:
        out = DeviceResult.empty(db.B, db.W, db.m.device)
    r = out.struct()
    _check(L.gr_solve(C.byref(b), strategy, C.byref(r), _ptr(fell_back), _ptr(ws), ws.numel(),
                      _stream(stream)), "gr_solve")
    return out


# ---- sharded exact solving ---------------------------------------------------
class ExactSession:
    """Step-wise exact solve (prepare / level / finish) for multi-GPU drivers."""

    def __init__(self, db: DeviceBatch, which: int, out: Optional[DeviceResult] = None,
                 stream=None):
        self.L = lib()
        self.db, self.which = db, which
        self.b = db.struct(which == PMS)
        nbytes = self.L.gr_workspace_bytes(C.byref(self.b), which)
        if nbytes == 0:
            raise GrError("gr_workspace_bytes rejected the batch")
        self.ws = workspace(nbytes, db.m.device, tag=f"session{which}")
        self.out = out if out is not None else DeviceResult.empty(db.B, db.W, db.m.device)
        self.r = self.out.struct()
        self.stream = stream

    def prepare(self) -> int:
        """Pack + plan level 1; returns the number of instances still searching."""
        n = C.c_int32(0)
        _check(self.L.gr_exact_prepare(C.byref(self.b), self.which, C.byref(self.r),
                                       _ptr(self.ws), self.ws.numel(), _stream(self.stream),
                                       C.byref(n)), "gr_exact_prepare")
        return int(n.value)

    def level(self, k: int, shard: int = 0, nshard: int = 1):
        _check(self.L.gr_exact_level(C.byref(self.b), self.which, k, shard, nshard, _ptr(self.ws),
                                     self.ws.numel(), _stream(self.stream)), "gr_exact_level")

    def level_keys(self):
        """torch int64 view [B] of the per-instance level keys (for all_reduce MIN)."""
        torch = _torch()
        p = self.L.gr_exact_level_keys(C.byref(self.b), self.which, _ptr(self.ws))
        base = _ptr(self.ws)
        off = (p - base) // 1
        return self.ws[off: off + 8 * self.db.B].view(torch.int64)

    def finish(self, k: int) -> int:
        n = C.c_int32(0)
        _check(self.L.gr_exact_finish(C.byref(self.b), self.which, k, C.byref(self.r),
                                      _ptr(self.ws), self.ws.numel(), _stream(self.stream),
                                      C.byref(n)), "gr_exact_finish")
        return int(n.value)


# ---- greedy at scale ---------------------------------------------------------
class PairSession:
    """Step-wise fused PMS + MHS (gr_pair_prepare / level / finish) for the
    rank-range-sharded driver: same protocol as ExactSession, but level_keys()
    returns both key arrays (PMS, MHS) to all-reduce."""

    def __init__(self, db: DeviceBatch, out_pms: Optional[DeviceResult] = None,
                 out_mhs: Optional[DeviceResult] = None, stream=None):
        self.L = lib()
        self.db = db
        self.b = db.struct(False)
        nbytes = self.L.gr_workspace_bytes(C.byref(self.b), PMS)
        if nbytes == 0:
            raise GrError("gr_workspace_bytes rejected the batch")
        half = (nbytes + 255) // 256 * 256
        self.ws = workspace(2 * half, db.m.device, tag="pair_session")
        dev = db.m.device
        self.out_pms = out_pms if out_pms is not None else DeviceResult.empty(db.B, db.W, dev)
        self.out_mhs = out_mhs if out_mhs is not None else DeviceResult.empty(db.B, db.W, dev)
        self.r1, self.r2 = self.out_pms.struct(), self.out_mhs.struct()
        self.stream = stream

    def prepare(self) -> int:
        n = C.c_int32(0)
        _check(self.L.gr_pair_prepare(C.byref(self.b), C.byref(self.r1), C.byref(self.r2),
                                      _ptr(self.ws), self.ws.numel(), _stream(self.stream),
                                      C.byref(n)), "gr_pair_prepare")
        return int(n.value)

    def level(self, k: int, shard: int = 0, nshard: int = 1):
        _check(self.L.gr_pair_level(C.byref(self.b), k, shard, nshard, _ptr(self.ws),
                                    self.ws.numel(), _stream(self.stream)), "gr_pair_level")

    def level_keys(self):
        """(PMS keys, MHS keys): torch int64 views [B] of the workspace."""
        torch = _torch()
        base = _ptr(self.ws)
        out = []
        for which in (0, 1):
            p = self.L.gr_pair_level_keys(C.byref(self.b), _ptr(self.ws), which)
            off = p - base
            out.append(self.ws[off: off + 8 * self.db.B].view(torch.int64))
        return tuple(out)

    def finish(self, k: int) -> int:
        n = C.c_int32(0)
        _check(self.L.gr_pair_finish(C.byref(self.b), k, C.byref(self.r1), C.byref(self.r2),
                                     _ptr(self.ws), self.ws.numel(), _stream(self.stream),
                                     C.byref(n)), "gr_pair_finish")
        return int(n.value)


def bitmatrix_ld(n_pos: int) -> int:
    return int(lib().gr_bitmatrix_ld(n_pos))


@dataclass
class DeviceBitMatrix:
    m: int
    n_pos: int
    ld: int
    bits: "object"  # int64 [m, ld]
    n_neg: int
    neg: "object"  # int64 [n_neg, ceil(m/64)] or None
    bad: int = 0  # 1: id out of range, 2: empty positive clause, 4: repeated id in a clause
    pos_off: "object" = None  # device CSR of phi+ (enables the incremental greedy)
    pos_var: "object" = None
    w: "object" = None  # optional int32 view of uint32 weights [m] (weighted mhs, f4)

    def struct(self) -> GrBitmatrix:
        vb = 0 if self.pos_var is None else self.pos_var.element_size()
        return GrBitmatrix(self.m, self.n_pos, self.ld, _ptr(self.bits), self.n_neg,
                           _ptr(self.neg), _ptr(self.pos_off), _ptr(self.pos_var), vb,
                           _ptr(self.w))


def pack_bitmatrix(m, pos_off, pos_var, neg_off, neg_var, device="cuda", stream=None,
                   check: bool = True, keep_csr: bool = True) -> DeviceBitMatrix:
    """Device clause packing (a1): CSR variable lists -> var-major phi+ bits and
    clause-major phi- masks (gr_pack_varmajor / gr_pack_clausemajor).  The
    CSR tensors may be host (numpy) or device (torch) arrays."""
    torch = _torch()
    L = lib()

    def dev(a, dt):
        if isinstance(a, np.ndarray):
            return torch.from_numpy(np.ascontiguousarray(a)).to(device)
        return a.to(device)

    po, pv = dev(pos_off, np.int64), dev(pos_var, None)
    no, nv = dev(neg_off, np.int64), dev(neg_var, None)
    n_pos, n_neg = int(po.numel() - 1), int(no.numel() - 1)
    ld = bitmatrix_ld(n_pos)
    # the tiled device pack writes every word (no clearing pass)
    bits = torch.empty((m, ld), dtype=torch.int64, device=device)
    mw = (m + 63) // 64
    neg = torch.zeros((max(n_neg, 1), mw), dtype=torch.int64, device=device)
    bad = torch.zeros(1, dtype=torch.int32, device=device)
    st = _stream(stream)
    _check(L.gr_pack_varmajor(m, n_pos, _ptr(po), _ptr(pv), pv.element_size(), _ptr(bits), ld,
                              _ptr(bad), st), "gr_pack_varmajor")
    badn = torch.zeros(1, dtype=torch.int32, device=device)
    _check(L.gr_pack_clausemajor(m, n_neg, _ptr(no), _ptr(nv), nv.element_size(), _ptr(neg),
                                 _ptr(badn), st), "gr_pack_clausemajor")
    b = int(bad.item()) if check else 0
    b |= int(badn.item()) & 1 if check else 0
    return DeviceBitMatrix(m, n_pos, ld, bits, n_neg, neg if n_neg else None, b,
                           po if keep_csr else None, pv if keep_csr else None)


def greedy_matrix_workspace_bytes(bm: DeviceBitMatrix) -> int:
    s = bm.struct()
    return int(lib().gr_greedy_matrix_workspace_bytes(C.byref(s)))


@dataclass
class GreedyMatrixResult:
    assign: "object"  # int64 [ceil(m/64)]
    status: "object"  # int32 [1]
    picks: "object"   # int32 [m]
    n_picks: int


def mhs_greedy_matrix(bm: DeviceBitMatrix, stream=None) -> GreedyMatrixResult:
    """(c) at scale: greedy mhs over the bit matrix (gr_mhs_greedy_matrix)."""
    torch = _torch()
    L = lib()
    s = bm.struct()
    nbytes = L.gr_greedy_matrix_workspace_bytes(C.byref(s))
    if nbytes == 0:
        raise GrError("gr_greedy_matrix_workspace_bytes rejected the matrix")
    ws = workspace(nbytes, bm.bits.device, tag="greedy_matrix")
    dev = bm.bits.device
    assign = torch.zeros((bm.m + 63) // 64, dtype=torch.int64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    picks = torch.full((bm.m,), -1, dtype=torch.int32, device=dev)
    n = C.c_int32(0)
    _check(L.gr_mhs_greedy_matrix(C.byref(s), _ptr(assign), _ptr(status), _ptr(picks), C.byref(n),
                                  _ptr(ws), ws.numel(), _stream(stream)), "gr_mhs_greedy_matrix")
    return GreedyMatrixResult(assign, status, picks, int(n.value))


class GrClauseLists(C.Structure):
    _fields_ = [("m", C.c_int32), ("n_pos", C.c_int64), ("nnz", C.c_int64),
                ("pos_off", C.c_void_p), ("pos_var", C.c_void_p), ("var_bytes", C.c_int32),
                ("n_neg", C.c_int32), ("neg", C.c_void_p), ("w", C.c_void_p)]


def mhs_greedy_lists(m, pos_off, pos_var, neg_off, neg_var, w=None, device="cuda", stream=None,
                     nnz=None) -> GreedyMatrixResult:
    """(c) at scale from clause lists alone (gr_mhs_greedy_lists, f3): phi-
    packed to clause-major masks on the device (gr_pack_clausemajor), then the
    greedy over the variable -> clause lists built on the device.  CSR arrays
    may be host (numpy) or device (torch); ``nnz`` = pos_off[-1] (read from
    the host array when not given); w: device int32 view of uint32 [m]."""
    torch = _torch()
    L = lib()

    def dev(a):
        if isinstance(a, np.ndarray):
            return torch.from_numpy(np.ascontiguousarray(a)).to(device)
        return a.to(device)

    if nnz is None:
        nnz = int(pos_off[-1])
    po, pv, no, nv = dev(pos_off), dev(pos_var), dev(neg_off), dev(neg_var)
    if pv.data_ptr() % 16:  # the C-ABI reads pos_var in aligned 16-byte groups
        pv = pv.clone()
    n_pos, n_neg = int(po.numel() - 1), int(no.numel() - 1)
    mw = (m + 63) // 64
    neg = torch.zeros((max(n_neg, 1), mw), dtype=torch.int64, device=device)
    st = _stream(stream)
    if n_neg:
        _check(L.gr_pack_clausemajor(m, n_neg, _ptr(no), _ptr(nv), nv.element_size(), _ptr(neg),
                                     None, st), "gr_pack_clausemajor")
    s = GrClauseLists(m, n_pos, int(nnz), _ptr(po), _ptr(pv), pv.element_size(), n_neg,
                      _ptr(neg) if n_neg else None, _ptr(w))
    nbytes = L.gr_greedy_lists_workspace_bytes(C.byref(s))
    if nbytes == 0:
        raise GrError("gr_greedy_lists_workspace_bytes rejected the lists: " + lib().gr_last_error().decode())
    ws = workspace(nbytes, po.device, tag="greedy_lists")
    assign = torch.zeros(mw, dtype=torch.int64, device=po.device)
    status = torch.zeros(1, dtype=torch.int32, device=po.device)
    picks = torch.full((m,), -1, dtype=torch.int32, device=po.device)
    n = C.c_int32(0)
    _check(L.gr_mhs_greedy_lists(C.byref(s), _ptr(assign), _ptr(status), _ptr(picks), C.byref(n),
                                 _ptr(ws), ws.numel(), st), "gr_mhs_greedy_lists")
    return GreedyMatrixResult(assign, status, picks, int(n.value))


def greedy_count_shard(bm: DeviceBitMatrix, U, counts, stream=None):
    """counts[v] = |{c in this shard : U[c] and v in c}| (gr_greedy_count_shard)."""
    s = bm.struct()
    _check(lib().gr_greedy_count_shard(C.byref(s), _ptr(U), _ptr(counts), _stream(stream)),
           "gr_greedy_count_shard")


class GreedyShard:
    """One rank's column shard of the greedy (gr_greedy_shard_*, SURVEY.md
    §8(e) C5).  Argument marshalling only: begin/step/state/private/remove/
    finalize map one-to-one onto the C-ABI; the exchange between steps is the
    caller's (multigpu.greedy_matrix_sharded)."""

    def __init__(self, bm: DeviceBitMatrix, stream=None):
        torch = _torch()
        self.L, self.bm, self.stream = lib(), bm, stream
        self.s = bm.struct()
        nbytes = self.L.gr_greedy_shard_workspace_bytes(C.byref(self.s))
        if nbytes == 0:
            raise GrError("gr_greedy_shard_workspace_bytes rejected the shard")
        dev = bm.bits.device
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.counts = torch.zeros(bm.m, dtype=torch.int32, device=dev)  # uint32 counts

    def begin(self):
        _check(self.L.gr_greedy_shard_begin(C.byref(self.s), _ptr(self.counts), _ptr(self.ws),
                                            self.ws.numel(), _stream(self.stream)),
               "gr_greedy_shard_begin")

    def step(self):
        _check(self.L.gr_greedy_shard_step(C.byref(self.s), _ptr(self.counts), _ptr(self.ws),
                                           self.ws.numel(), _stream(self.stream)),
               "gr_greedy_shard_step")

    def state(self, picks=None):
        n, d = C.c_int32(0), C.c_int32(0)
        _check(self.L.gr_greedy_shard_state(C.byref(self.s), _ptr(self.ws), self.ws.numel(),
                                            C.byref(n), C.byref(d),
                                            _ptr(picks) if picks is not None else None,
                                            _stream(self.stream)), "gr_greedy_shard_state")
        return int(n.value), bool(d.value)

    def private(self, only, flags):
        _check(self.L.gr_greedy_shard_private(C.byref(self.s), int(only), _ptr(flags),
                                              _ptr(self.ws), self.ws.numel(),
                                              _stream(self.stream)), "gr_greedy_shard_private")

    def remove(self, j):
        _check(self.L.gr_greedy_shard_remove(C.byref(self.s), int(j), _ptr(self.ws),
                                             self.ws.numel(), _stream(self.stream)),
               "gr_greedy_shard_remove")

    def finalize(self, removed, assign, status):
        _check(self.L.gr_greedy_shard_finalize(C.byref(self.s), _ptr(removed), _ptr(assign),
                                               _ptr(status), _ptr(self.ws), self.ws.numel(),
                                               _stream(self.stream)), "gr_greedy_shard_finalize")


def version() -> str:
    return lib().gr_version().decode()


# ---- launch accounting / profiling ---------------------------------------------
def launch_count() -> int:
    """Kernel launches made by libgrsolve since it was loaded."""
    return int(lib().gr_launch_count())


class Profiler:
    """gr_profile(mode): 1 = CUDA-event duration of every launch (on its own
    stream), 2 = also the enumeration kernel's work-counting instantiation."""

    def __init__(self, mode: int = 1):
        self.mode = mode

    def start(self):
        _check(lib().gr_profile(self.mode), "gr_profile")
        return self

    def read(self) -> dict:
        arr = (GrKernelStat * 64)()
        n = lib().gr_profile_read(C.cast(arr, C.c_void_p), 64)
        out = {}
        for i in range(n):
            st = arr[i]
            out[st.name.decode()] = {"launches": int(st.launches), "ms": float(st.ms),
                                     "work": [int(x) for x in st.work]}
        return out

    def stop(self) -> dict:
        r = self.read()
        lib().gr_profile(0)
        return r


def profiler(mode: int = 1) -> Profiler:
    return Profiler(mode)
