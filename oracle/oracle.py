"""ctypes front end of the CPU oracle (oracle/hb_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, always as the checker or the
timed CPU baseline, never as part of the product path.

`run_oracle` restates the reference driver loop (engine.py:330-435 with a
CentralityAccumulator observer, centrality.py:104-171) on top of the C
restatement of the kernels, and can record per-iteration digests so tests can
compare registers, estimates and changed counts iteration by iteration.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liborc.so")
_lib = None

_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_int = ctypes.c_int
_dbl = ctypes.c_double
_vp = ctypes.c_void_p


def build() -> str:
    """Compile liborc.so in place (make); returns its path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_mix64.restype = _u64
        L.orc_mix64.argtypes = [_u64]
        L.orc_hash.restype = _u64
        L.orc_hash.argtypes = [_u64, _u64, _u64]
        L.orc_hash_items.restype = None
        L.orc_hash_items.argtypes = [_i64, _vp, _vp, _u64, _vp]
        L.orc_alpha.restype = _dbl
        L.orc_alpha.argtypes = [_i64]
        L.orc_constants.restype = None
        L.orc_constants.argtypes = [_int, _vp, _vp, _vp]
        L.orc_estimate_row.restype = _dbl
        L.orc_estimate_row.argtypes = [_vp, _i64, _dbl, _dbl, _dbl]
        L.orc_estimate_rows.restype = None
        L.orc_estimate_rows.argtypes = [_vp, _i64, _i64, _int, _vp]
        L.orc_seed.restype = None
        L.orc_seed.argtypes = [_i64, _int, _int, _u64, _vp, _vp, _vp]
        L.orc_union_range.restype = _i64
        L.orc_union_range.argtypes = [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                      _int, _int]
        L.orc_iterate_mt.restype = _i64
        L.orc_iterate_mt.argtypes = [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _int,
                                     _int, _int]
        L.orc_iterate_range_mt.restype = _i64
        L.orc_iterate_range_mt.argtypes = [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                           _int, _int, _int]
        L.orc_accumulate.restype = None
        L.orc_accumulate.argtypes = [_i64, _i64, _vp, _vp, _vp, _vp]
        L.orc_finalize.restype = None
        L.orc_finalize.argtypes = [_i64, _vp, _vp, _vp, _vp, _vp, _vp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# -- scalar helpers (hll.py) -------------------------------------------------

def hash_items(items, replicas, seed: int) -> np.ndarray:
    items = _c(items, np.uint64)
    replicas = _c(np.broadcast_to(np.asarray(replicas, np.uint64), items.shape), np.uint64)
    out = np.empty(items.shape, np.uint64)
    lib().orc_hash_items(items.size, _p(items), _p(replicas), seed & ((1 << 64) - 1), _p(out))
    return out


def constants(b: int):
    a2, lc, pf = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    lib().orc_constants(b, ctypes.byref(a2), ctypes.byref(lc), ctypes.byref(pf))
    return a2.value, lc.value, pf.value


def estimate_rows(regs: np.ndarray, b: int) -> np.ndarray:
    regs = _c(regs, np.uint8)
    n = regs.shape[0]
    out = np.zeros(n, np.float64)
    if n:
        lib().orc_estimate_rows(_p(regs), 0, n, b, _p(out))
    return out


def seed_registers(n: int, b: int, width: int = 5, seed: int = 0, weights=None):
    regs = np.zeros((n, 1 << b), np.uint8)
    est = np.zeros(n, np.float64)
    w = None if weights is None else _c(weights, np.int64)
    lib().orc_seed(n, b, width, seed & ((1 << 64) - 1), None if w is None else _p(w),
                   _p(regs), _p(est))
    return regs, est


def union_pass(offsets, succ, cur, chg_prev, est, b: int, skip: bool = True,
               workers: int = 1, lo: int | None = None, hi: int | None = None):
    """One hll_union_range pass (all nodes, or [lo, hi) single-threaded).

    Returns (nch, nxt, chg_now, new_est); rows outside [lo, hi) of the outputs are
    left zero.
    """
    offsets = _c(offsets, np.int64)
    succ = _c(succ, np.int64)
    cur = _c(cur, np.uint8)
    chg_prev = _c(chg_prev, np.uint8)
    est = _c(est, np.float64)
    n = offsets.shape[0] - 1
    nxt = np.zeros_like(cur)
    chg_now = np.zeros(n, np.uint8)
    new_est = np.zeros(n, np.float64)
    if lo is None and hi is None:
        nch = lib().orc_iterate_mt(n, _p(offsets), _p(succ), _p(cur), _p(nxt), _p(chg_prev),
                                   _p(chg_now), _p(est), _p(new_est), b, int(skip), workers)
    else:
        lo = 0 if lo is None else lo
        hi = n if hi is None else hi
        nch = lib().orc_union_range(lo, hi, _p(offsets), _p(succ), _p(cur), _p(nxt),
                                    _p(chg_prev), _p(chg_now), _p(est), _p(new_est), b,
                                    int(skip))
    return int(nch), nxt, chg_now, new_est


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@dataclass
class OracleResult:
    t: int
    registers: np.ndarray
    est: np.ndarray
    sum_dist: np.ndarray
    sum_recip: np.ndarray
    coreach: np.ndarray
    closeness: np.ndarray
    harmonic: np.ndarray
    lin: np.ndarray
    nch: list = field(default_factory=list)
    reg_digests: list = field(default_factory=list)
    est_digests: list = field(default_factory=list)
    snapshots: list = field(default_factory=list)


def run_oracle(offsets, succ, b: int, seed: int = 0, width: int = 5, workers: int = 1,
               skip: bool = True, max_iterations: int | None = None, weights=None,
               record: bool = True, keep_snapshots: bool = False,
               reg_digest=None) -> OracleResult:
    """engine.run(g, HyperBallConfig(CounterParams(b, width, seed)), [CentralityAccumulator])
    restated: initialize (engine.py:330-348), iterate until no counter changes
    (engine.py:413-435), accumulate per iteration (centrality.py:132-150), finalize
    (centrality.py:153-171).  Index 0 of the digest lists is the seeded state.
    reg_digest: digest function of the register matrix (default: sha256 of the bytes)."""
    rdig = reg_digest or sha
    offsets = _c(offsets, np.int64)
    succ = _c(succ, np.int64)
    n = offsets.shape[0] - 1
    cur, est = seed_registers(n, b, width, seed, weights)
    chg_prev = np.ones(n, np.uint8)
    sum_dist = np.zeros(n, np.float64)
    sum_recip = np.zeros(n, np.float64)
    res = OracleResult(0, cur, est, sum_dist, sum_recip, None, None, None, None)
    if record:
        res.reg_digests.append(rdig(cur))
        res.est_digests.append(sha(est))
    if keep_snapshots:
        res.snapshots.append((cur.copy(), est.copy(), chg_prev.copy()))
    t = 0
    if n > 0:
        while True:
            nch, nxt, chg_now, new_est = union_pass(offsets, succ, cur, chg_prev, est, b, skip,
                                                    workers)
            t += 1
            lib().orc_accumulate(n, t, _p(est), _p(new_est), _p(sum_dist), _p(sum_recip))
            cur, est, chg_prev = nxt, new_est, chg_now
            res.nch.append(nch)
            if record:
                res.reg_digests.append(rdig(cur))
                res.est_digests.append(sha(est))
            if keep_snapshots:
                res.snapshots.append((cur.copy(), est.copy(), chg_prev.copy()))
            if nch == 0:
                break
            if max_iterations is not None and t >= max_iterations:
                raise RuntimeError(f"max_iterations reached at t={t} with {nch} changing")
    coreach = est.astype(np.float64).copy()
    clo = np.zeros(n)
    har = np.zeros(n)
    lin = np.zeros(n)
    if n:
        lib().orc_finalize(n, _p(sum_dist), _p(sum_recip), _p(coreach), _p(clo), _p(har),
                           _p(lin))
    res.t, res.registers, res.est = t, cur, est
    res.coreach, res.closeness, res.harmonic, res.lin = coreach, clo, har, lin
    return res


def exact_union_pass(offsets, succ, cur, chg_prev, est, weights, skip: bool = True):
    """One bitset_union_range pass over all nodes (_kernels.py:133-172), vectorised:
    a node is active when it or one of its in-neighbours changed; an active row is the OR
    of its own row and all its in-neighbours' rows; a changed row's estimate is the
    weighted popcount of its MSB-first bits (_kernels.py:117-130) as float."""
    offsets = _c(offsets, np.int64)
    succ = _c(succ, np.int64)
    n = offsets.shape[0] - 1
    nxt = cur.copy()
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(offsets))
    prev = np.asarray(chg_prev).astype(bool)
    act = prev.copy()
    if succ.size:
        np.logical_or.at(act, rows, prev[succ])
    sel = act[rows] if skip else np.ones(rows.shape, bool)
    if sel.any():
        np.bitwise_or.at(nxt, rows[sel], cur[succ[sel]])
    changed = (nxt != cur).any(axis=1) if n else np.zeros(0, bool)
    new_est = est.copy()
    if changed.any():
        bits = np.unpackbits(nxt[changed], axis=1)[:, :n].astype(np.int64)
        new_est[changed] = (bits @ np.asarray(weights, np.int64)).astype(np.float64)
    return int(changed.sum()), nxt, changed.astype(np.uint8), new_est


def run_exact_oracle(offsets, succ, weights=None, skip: bool = True,
                     record: bool = True) -> OracleResult:
    """engine.run with backend="exact" (engine.py:178-213) restated: seed one bit per
    node (engine.py:194-200), iterate exact_union_pass to convergence, accumulate and
    finalize as run_oracle."""
    offsets = _c(offsets, np.int64)
    n = offsets.shape[0] - 1
    w = np.ones(n, np.int64) if weights is None else _c(weights, np.int64)
    cur = np.zeros((n, (n + 7) // 8), np.uint8)
    v = np.arange(n)
    cur[v, v >> 3] |= (0x80 >> (v & 7)).astype(np.uint8)
    est = w.astype(np.float64)
    chg_prev = np.ones(n, np.uint8)
    sum_dist = np.zeros(n, np.float64)
    sum_recip = np.zeros(n, np.float64)
    res = OracleResult(0, cur, est, sum_dist, sum_recip, None, None, None, None)
    if record:
        res.reg_digests.append(sha(cur))
        res.est_digests.append(sha(est))
    t = 0
    if n > 0:
        while True:
            nch, nxt, chg_now, new_est = exact_union_pass(offsets, succ, cur, chg_prev, est,
                                                          w, skip)
            t += 1
            lib().orc_accumulate(n, t, _p(est), _p(new_est), _p(sum_dist), _p(sum_recip))
            cur, est, chg_prev = nxt, new_est, chg_now
            res.nch.append(nch)
            if record:
                res.reg_digests.append(sha(cur))
                res.est_digests.append(sha(est))
            if nch == 0:
                break
    coreach = est.copy()
    clo, har, lin = np.zeros(n), np.zeros(n), np.zeros(n)
    if n:
        lib().orc_finalize(n, _p(sum_dist), _p(sum_recip), _p(coreach), _p(clo), _p(har),
                           _p(lin))
    res.t, res.registers, res.est = t, cur, est
    res.coreach, res.closeness, res.harmonic, res.lin = coreach, clo, har, lin
    return res
