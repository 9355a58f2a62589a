"""CPU oracle for the GPURepair Solve step -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2011_08373_b200``) never imports it.  ``oracle.c`` holds every line
of arithmetic; this file only marshals numpy arrays through ctypes.

Status values (by meaning): SAT = 0, UNSAT = 1, SAT_NEG_VIOLATED = 2,
BADINPUT = 3.

Parity status: pinned (see tests/test_oracle.py and DESIGN.md §3): the exact
solvers against closed forms, the paper's worked example, an
independent 2^m brute force and Koenig's theorem; the greedy against hand
derivations and its defining invariants.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "oracle.c")

SAT, UNSAT, SAT_NEG_VIOLATED, BADINPUT = 0, 1, 2, 3
U64MAX = (1 << 64) - 1


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (-O2, OpenMP)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-Wall",
                               "-o", LIB, SRC])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        p = C.c_void_p
        L.or_num_threads.restype = C.c_int
        L.or_set_threads.argtypes = [C.c_int]
        L.or_pms.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, p, p, C.c_int, p, p, p, p]
        L.or_pms_kstart.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, p, C.c_int, C.c_int, p, p,
                                    p, p]
        L.or_pms_kstart.restype = C.c_int
        L.or_pms_brute.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, p, p, p, p, p]
        L.or_mhs.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, p, C.c_int, p, p, p, p]
        L.or_greedy.argtypes = [C.c_int, C.c_int64, p, p, C.c_int64, p, p, p, p, p, p, p]
        L.or_greedy_w.argtypes = [C.c_int, C.c_int64, p, p, C.c_int64, p, p, p, p, p, p, p, p]
        L.or_greedy_w.restype = C.c_int
        L.or_greedy_masks.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, p, p, p, p, p]
        L.or_greedy_masks_w.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, p, p, p, p, p, p]
        L.or_greedy_masks_w.restype = C.c_int
        L.or_batch.argtypes = [C.c_int, C.c_int, C.c_int, p, p, p, p, p, C.c_int, C.c_int,
                               p, p, p, p]
        L.or_min_feasible_product.argtypes = [C.c_int, p, p, C.c_int, C.c_int, p, p]
        L.or_min_feasible_product.restype = C.c_uint64
        L.or_feasible.argtypes = [C.c_uint64, C.c_int, C.c_int, p]
        for f in (L.or_pms, L.or_pms_brute, L.or_mhs, L.or_greedy, L.or_greedy_masks, L.or_batch):
            f.restype = C.c_int
        _lib = L
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def num_threads() -> int:
    return int(lib().or_num_threads())


def set_threads(t: int) -> None:
    lib().or_set_threads(int(t))


@dataclass
class Result:
    status: int  # -1: support of phi+ > 64 variables (no oracle value)
    assign: int  # mask (all W words joined); 0 when UNSAT
    cost: int  # U64MAX when UNSAT
    decided: int = 0


def _join(words) -> int:
    return sum(int(x) << (64 * i) for i, x in enumerate(words))


def _inst(masks, W):
    masks = np.ascontiguousarray(np.asarray(masks, np.uint64).reshape(-1, W))
    return masks


def pms(m: int, n_pos: int, masks, w=None, reduce: int = 1, W: int = 1) -> Result:
    """Exact PMS (w None) / WPMS of one instance; masks [n, W] positives first."""
    mk = _inst(masks, W)
    wa = None if w is None else np.ascontiguousarray(np.asarray(w, np.uint32))
    a, c, s, d = (np.zeros(W, np.uint64), np.zeros(1, np.uint64), np.zeros(1, np.int32),
                  np.zeros(1, np.uint64))
    rc = lib().or_pms(m, W, n_pos, mk.shape[0] - n_pos, _ptr(mk), _ptr(wa), reduce,
                      _ptr(a), _ptr(c), _ptr(s), _ptr(d))
    if rc:
        raise RuntimeError(f"or_pms failed: {rc}")
    return Result(int(s[0]), _join(a), int(c[0]), int(d[0]))


def pms_kstart(m: int, n_pos: int, masks, kstart: int, reduce: int = 1, W: int = 1) -> Result:
    """Unit-weight PMS enumerating levels >= kstart only (incremental Solve, f2)."""
    mk = _inst(masks, W)
    a, c, s, d = (np.zeros(W, np.uint64), np.zeros(1, np.uint64), np.zeros(1, np.int32),
                  np.zeros(1, np.uint64))
    rc = lib().or_pms_kstart(m, W, n_pos, mk.shape[0] - n_pos, _ptr(mk), reduce, kstart,
                             _ptr(a), _ptr(c), _ptr(s), _ptr(d))
    if rc:
        raise RuntimeError(f"or_pms_kstart failed: {rc}")
    return Result(int(s[0]), _join(a), int(c[0]), int(d[0]))


def pms_brute(m: int, n_pos: int, masks, w=None, W: int = 1) -> Result:
    """Independent 2^m scan (m <= 30), key (W, popcount, mask)."""
    mk = _inst(masks, W)
    wa = None if w is None else np.ascontiguousarray(np.asarray(w, np.uint32))
    a, c, s = np.zeros(1, np.uint64), np.zeros(1, np.uint64), np.zeros(1, np.int32)
    rc = lib().or_pms_brute(m, W, n_pos, mk.shape[0] - n_pos, _ptr(mk), _ptr(wa),
                            _ptr(a), _ptr(c), _ptr(s))
    if rc:
        raise RuntimeError(f"or_pms_brute failed: {rc}")
    return Result(int(s[0]), int(a[0]), int(c[0]))


def mhs(m: int, n_pos: int, masks, reduce: int = 1, W: int = 1) -> Result:
    mk = _inst(masks, W)
    a, c, s, d = (np.zeros(W, np.uint64), np.zeros(1, np.uint64), np.zeros(1, np.int32),
                  np.zeros(1, np.uint64))
    rc = lib().or_mhs(m, W, n_pos, mk.shape[0] - n_pos, _ptr(mk), reduce, _ptr(a), _ptr(c),
                      _ptr(s), _ptr(d))
    if rc:
        raise RuntimeError(f"or_mhs failed: {rc}")
    return Result(int(s[0]), _join(a), int(c[0]), int(d[0]))


@dataclass
class GreedyResult:
    status: int
    picks: np.ndarray  # pick order before pruning (0-based var ids)
    in_S: np.ndarray  # uint8 [m], final pruned set
    n_final: int


def greedy_csr(m, pos_off, pos_var, neg_off, neg_var, w=None) -> GreedyResult:
    """Greedy over CSR clause lists; with weights w the weighted (ratio) greedy."""
    pos_off = np.ascontiguousarray(pos_off, np.int64)
    pos_var = np.ascontiguousarray(pos_var, np.int32)
    neg_off = np.ascontiguousarray(neg_off, np.int64)
    neg_var = np.ascontiguousarray(neg_var, np.int32)
    picks = np.zeros(max(m, 1), np.int32)
    inS = np.zeros(max(m, 1), np.uint8)
    nu, nf, st = np.zeros(1, np.int32), np.zeros(1, np.int32), np.zeros(1, np.int32)
    if w is None:
        rc = lib().or_greedy(m, pos_off.shape[0] - 1, _ptr(pos_off), _ptr(pos_var),
                             neg_off.shape[0] - 1, _ptr(neg_off), _ptr(neg_var), _ptr(picks),
                             _ptr(nu), _ptr(inS), _ptr(nf), _ptr(st))
    else:
        wa = np.ascontiguousarray(np.asarray(w, np.uint32))
        rc = lib().or_greedy_w(m, pos_off.shape[0] - 1, _ptr(pos_off), _ptr(pos_var),
                               neg_off.shape[0] - 1, _ptr(neg_off), _ptr(neg_var), _ptr(wa),
                               _ptr(picks), _ptr(nu), _ptr(inS), _ptr(nf), _ptr(st))
    if rc:
        raise RuntimeError(f"or_greedy failed: {rc}")
    return GreedyResult(int(st[0]), picks[: int(nu[0])].copy(), inS[:m].copy(), int(nf[0]))


def greedy(m: int, n_pos: int, masks, W: int = 1, w=None):
    """Greedy mhs over mask-encoded clauses -> (status, assign words, picks);
    with weights w the weighted (ratio) greedy (f4)."""
    mk = _inst(masks, W)
    a = np.zeros(W, np.uint64)
    picks = np.zeros(max(m, 1), np.int32)
    nu, st = np.zeros(1, np.int32), np.zeros(1, np.int32)
    wa = None if w is None else np.ascontiguousarray(np.asarray(w, np.uint32))
    rc = lib().or_greedy_masks_w(m, W, n_pos, mk.shape[0] - n_pos, _ptr(mk), _ptr(wa), _ptr(a),
                                 _ptr(picks), _ptr(nu), _ptr(st))
    if rc:
        raise RuntimeError(f"or_greedy_masks failed: {rc}")
    return int(st[0]), a, picks[: int(nu[0])].copy()


@dataclass
class BatchResult:
    status: np.ndarray
    assign: np.ndarray  # [B, W]
    cost: np.ndarray
    decided: np.ndarray


def batch(which: str, cb, reduce: int = 1, weighted: bool = True) -> BatchResult:
    """Solve every instance of a synth.ClauseBatch: which in {pms, mhs, greedy, solve}
    (solve = composite mhs strategy with MaxSAT fallback; its ``decided`` holds
    the fallback flag)."""
    code = {"pms": 0, "mhs": 1, "greedy": 2, "solve": 3, "greedy_w": 4, "solve_w": 5}[which]
    W = cb.W
    B = cb.B
    assign = np.zeros((B, W), np.uint64)
    cost = np.zeros(B, np.uint64)
    status = np.zeros(B, np.int32)
    decided = np.zeros(B, np.uint64)
    m = np.ascontiguousarray(cb.m, np.int32)
    off = np.ascontiguousarray(cb.off, np.int64)
    npos = np.ascontiguousarray(cb.n_pos, np.int32)
    masks = np.ascontiguousarray(cb.masks, np.uint64)
    w = None
    ws = 0
    if weighted and cb.w is not None and which in ("pms", "solve", "greedy_w", "solve_w"):
        w = np.ascontiguousarray(cb.w, np.uint32)
        ws = w.shape[1]
    rc = lib().or_batch(code, B, W, _ptr(m), _ptr(off), _ptr(npos), _ptr(masks), _ptr(w), ws,
                        reduce, _ptr(assign), _ptr(cost), _ptr(status), _ptr(decided))
    if rc:
        raise RuntimeError(f"or_batch failed: {rc}")
    return BatchResult(status, assign, cost, decided)


def min_feasible_product(groups, n_pos: int, masks):
    """P15 helper: (count of feasible one-per-group sets, min feasible mask)."""
    goff = np.zeros(len(groups) + 1, np.int64)
    bits = []
    for g, grp in enumerate(groups):
        for v in grp:
            bits.append(1 << int(v))
        goff[g + 1] = len(bits)
    gbits = np.asarray(bits, np.uint64)
    mk = np.ascontiguousarray(np.asarray(masks, np.uint64).reshape(-1))
    best = np.zeros(1, np.uint64)
    n = lib().or_min_feasible_product(len(groups), _ptr(goff), _ptr(gbits), n_pos,
                                      mk.shape[0] - n_pos, _ptr(mk), _ptr(best))
    return int(n), int(best[0])


def feasible(x: int, n_pos: int, masks) -> bool:
    mk = np.ascontiguousarray(np.asarray(masks, np.uint64).reshape(-1))
    return bool(lib().or_feasible(x, n_pos, mk.shape[0] - n_pos, _ptr(mk)))
