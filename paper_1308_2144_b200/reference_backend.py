"""A backend for the reference engine's own loop (engine.py:138-175 protocol).

The reference's ``iterate`` (engine.py:362-399) drives a backend object through four
methods -- ``seed(weights, est)``, ``union_range(lo, hi, offsets, successors,
changed_prev, changed_now, est, new_est, skip_stable) -> int``, ``swap()``,
``counters()`` -- and hands numpy arrays to its observers.  ``CudaBackend`` implements that
protocol on the sm_100a kernels through the C-ABI, so a maintainer can register it next to
``_ProbabilisticBackend`` and keep the rest of the reference engine,
its observers and its CLI unchanged.  The registers stay on the device; only the arrays
the protocol exchanges cross PCIe (est / flags, O(n) per iteration).

This is the integration shim; the drop-in API in ``engine.py`` is the fast path (it keeps
estimates and accumulators on the device too).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .hll import CounterArray, estimator_constants, lc_table
from .schedule import build_schedule


class CudaBackend:
    """engine.py:138-175 backend protocol over hb_seed / hb_union_step.

    Constructed like the reference's ``_ProbabilisticBackend(n, params)``
    (engine.py:342-345); the graph arrives with the first ``union_range`` call (the
    reference passes ``offsets`` / ``successors`` to every call), so the schedule is built
    then -- or up front when ``graph`` is given.

    Worker ranges (engine.py:351-390): the reference's ``iterate`` splits [0, n) into
    arc-balanced ranges and calls ``union_range`` once per range from a thread pool, then
    ``swap()``.  The first call of an iteration (under a lock) runs the whole step on the
    device and keeps host copies of the new estimates and change flags; every call --
    the first included -- then writes only ITS rows of ``new_est`` / ``changed_now``
    (the reference kernel's contract, _kernels.py:3-6) and returns its rows' changed
    count, so the counts sum to the step's total for any worker count."""

    kind = "probabilistic"

    def __init__(self, n: int, params, graph=None, device=None, schedule: str = "auto"):
        import threading
        self.params, self.n = params, n
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.stream = torch.cuda.current_stream(self.device)
        self.order = schedule
        p = params.p
        dv = self.device
        self._cur = torch.zeros((n, p), dtype=torch.uint8, device=dv)
        self._nxt = torch.empty_like(self._cur)
        words = max((n + 31) // 32, 1)
        self.bits = [torch.zeros(words, dtype=torch.int32, device=dv) for _ in range(2)]
        self.est = torch.zeros(n, dtype=torch.float64, device=dv)
        self.lc = torch.from_numpy(lc_table(p)).to(dv)
        self.alpha_p2, self.lc_cut, _ = estimator_constants(p)
        self.counts = torch.zeros(2, dtype=torch.int64, device=dv)
        self.ticket = torch.zeros(1, dtype=torch.int64, device=dv)
        self.t = 0
        self.sched = None
        self._lock = threading.Lock()
        self._step = None          # (new_est host, changed_now host) of the running iteration
        if graph is not None:
            self._bind(graph.offsets, graph.successors)

    def _bind(self, offsets, successors) -> None:
        """Build the schedule; rows seeded in original order move to internal order."""
        self.sched = build_schedule(offsets, successors, self.params.b, self.device,
                                    self.order, stream=self.stream)
        if self.sched.perm is not None:
            self._cur = self.sched.to_internal(self._cur).contiguous()
            self.est = self.sched.to_internal(self.est).contiguous()

    # -- protocol --------------------------------------------------------------
    def seed(self, weights, est: np.ndarray) -> None:
        w = None
        if weights is not None:
            w = torch.from_numpy(np.asarray(getattr(weights, "values", weights),
                                            dtype=np.int64)).to(self.device)
        perm = self.sched.perm if self.sched is not None else None
        _lib.check(_lib.hb().hb_seed(
            self._cur.data_ptr(), self.est.data_ptr(), self.n, self.params.b,
            self.params.register_width, self.params.seed & ((1 << 64) - 1),
            perm.data_ptr() if perm is not None else None,
            w.data_ptr() if w is not None else None, self.lc.data_ptr(), self.alpha_p2,
            self.lc_cut, self.stream.cuda_stream), "hb_seed")
        if self.n:
            est[:] = self._to_original(self.est).cpu().numpy()

    def _to_original(self, x):
        return x if self.sched is None else self.sched.to_original(x)

    def union_range(self, lo, hi, offsets, successors, changed_prev, changed_now, est,
                    new_est, skip_stable) -> int:
        """Rows [lo, hi) of one iteration; any partition of [0, n) into worker ranges."""
        if not (0 <= lo <= hi <= self.n):
            raise ValueError(f"union_range: bad range [{lo}, {hi}) for n={self.n}")
        with self._lock:
            if self._step is None:
                self._step = self._full_step(offsets, successors, changed_prev, est,
                                             skip_stable)
            full_est, full_chg = self._step
        new_est[lo:hi] = full_est[lo:hi]
        changed_now[lo:hi] = full_chg[lo:hi]
        return int(np.count_nonzero(full_chg[lo:hi]))

    def _full_step(self, offsets, successors, changed_prev, est, skip_stable):
        if self.sched is None:
            self._bind(offsets, successors)
        self.t += 1
        s = self.sched
        prev = torch.from_numpy(np.packbits(np.asarray(changed_prev, dtype=bool),
                                            bitorder="little"))
        prev_dev = torch.zeros_like(self.bits[0]).view(torch.uint8)
        prev_dev[:prev.numel()].copy_(prev.to(self.device))
        prev_bits = s.to_internal_bits(prev_dev.view(torch.int32), self.n)
        self.est.copy_(s.to_internal(torch.from_numpy(np.ascontiguousarray(est)).to(self.device)))
        dense = (not skip_stable) or bool(np.all(changed_prev))
        # the recycled buffer must hold the current rows for the lazy write (a fresh
        # backend's nxt is uninitialised, and the reference's changed_prev may be
        # anything): refresh it from cur on the first step
        if self.t == 1:
            self._nxt.copy_(self._cur)
        _lib.union_step(_lib.StepArgs(
            n=self.n, lo=s.light_lo, hi=s.light_hi, offsets=s.offsets.data_ptr(),
            succ=s.succ.data_ptr(), cur=self._cur.data_ptr(), nxt=self._nxt.data_ptr(),
            chg_prev=prev_bits.data_ptr(), chg_now=self.bits[1].data_ptr(),
            est=self.est.data_ptr(), b=self.params.b, dense=int(dense), clear_chg_now=1,
            t=self.t, lc_table=self.lc.data_ptr(), alpha_p2=self.alpha_p2,
            lc_cut=self.lc_cut, nch_out=self.counts.data_ptr(),
            merged_out=self.counts.data_ptr() + 8, ticket=self.ticket.data_ptr(),
            stream=self.stream.cuda_stream, **_lib.schedule_args(s)))
        new = s.to_original(self.est).cpu().numpy()
        chg = s.to_original_bits(self.bits[1], self.n).cpu().numpy()
        return new, chg

    def swap(self) -> None:
        with self._lock:
            self._cur, self._nxt = self._nxt, self._cur
            self._step = None

    @property
    def cur(self) -> np.ndarray:
        """Host copy of the rows in original order (what the reference's
        HyperBallState.register_matrix / save read from backend.cur)."""
        return self.register_matrix()

    @property
    def nxt(self) -> np.ndarray:
        return self._to_original(self._nxt).cpu().numpy()

    def counters(self) -> CounterArray:
        return CounterArray.from_dense(self.register_matrix(), self.params)

    def register_matrix(self) -> np.ndarray:
        return self._to_original(self._cur).cpu().numpy()


def _flags_to_bits(flags, n: int, words: int, device) -> torch.Tensor:
    packed = torch.from_numpy(np.packbits(np.asarray(flags, dtype=bool), bitorder="little"))
    out = torch.zeros(words * 4, dtype=torch.uint8, device=device)
    out[:packed.numel()].copy_(packed.to(device))
    return out.view(torch.int32)


def _bits_to_flags(words: torch.Tensor, n: int) -> np.ndarray:
    b = np.unpackbits(words.view(torch.uint8).cpu().numpy(), bitorder="little")
    return b[:n].astype(bool)


class CudaExactBackend:
    """engine.py:178-213 _ExactBackend protocol over hb_exact_seed / hb_exact_union_step:
    one bitset row of n bits per node on the device (rows padded to a 16-byte stride)."""

    kind = "exact"

    def __init__(self, n: int, params, weights, graph, device=None):
        self.params, self.n = params, n
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.stream = torch.cuda.current_stream(self.device)
        dv = self.device
        self.offsets = torch.from_numpy(np.array(graph.offsets, dtype=np.int64)).to(dv)
        self.succ = torch.from_numpy(np.array(graph.successors, dtype=np.int32)).to(dv)
        self.row_bytes = (n + 7) // 8
        self.row_stride = max(16, (self.row_bytes + 15) // 16 * 16)
        self._cur = torch.zeros((n, self.row_stride), dtype=torch.uint8, device=dv)
        self._nxt = torch.zeros_like(self._cur)
        vals = getattr(weights, "values", weights)
        self.weights = (np.ones(n, dtype=np.int64) if vals is None
                        else np.ascontiguousarray(vals, dtype=np.int64))
        self._w = None if vals is None else torch.from_numpy(self.weights.copy()).to(dv)
        self.words = max((n + 31) // 32, 1)
        self.est = torch.zeros(n, dtype=torch.float64, device=dv)
        self.chg_now = torch.zeros(self.words, dtype=torch.int32, device=dv)
        self.counts = torch.zeros(2, dtype=torch.int64, device=dv)
        self.ticket = torch.zeros(1, dtype=torch.int64, device=dv)
        self.t = 0

    def seed(self, weights, est: np.ndarray) -> None:
        _lib.check(_lib.hb().hb_exact_seed(
            self.n, self.row_stride, self._cur.data_ptr(), self.est.data_ptr(),
            self._w.data_ptr() if self._w is not None else None, self.stream.cuda_stream),
            "hb_exact_seed")
        if self.n:
            est[:] = self.est.cpu().numpy()

    def union_range(self, lo, hi, offsets, successors, changed_prev, changed_now, est,
                    new_est, skip_stable) -> int:
        """One call per iteration over [0, n) (use workers=1 with this backend)."""
        if (lo, hi) != (0, self.n):
            raise ValueError("CudaExactBackend processes the whole graph per call (workers=1)")
        self.t += 1
        prev = _flags_to_bits(changed_prev, self.n, self.words, self.device)
        self.est.copy_(torch.from_numpy(np.ascontiguousarray(est)).to(self.device))
        dense = (not skip_stable) or bool(np.all(changed_prev))
        _lib.check(_lib.hb().hb_exact_union_step(
            self.n, self.offsets.data_ptr(), self.succ.data_ptr(), self._cur.data_ptr(),
            self._nxt.data_ptr(), self.row_stride, prev.data_ptr(), self.chg_now.data_ptr(),
            self.est.data_ptr(), None, None, self.t, int(dense),
            self._w.data_ptr() if self._w is not None else None, None, 0, 0, None, 0,
            self.counts.data_ptr(), self.counts.data_ptr() + 8, self.stream.cuda_stream),
            "hb_exact_union_step")
        new_est[:] = self.est.cpu().numpy()
        changed_now[:] = _bits_to_flags(self.chg_now, self.n)
        return int(self.counts[0].item())

    def swap(self) -> None:
        self._cur, self._nxt = self._nxt, self._cur

    @property
    def cur(self) -> np.ndarray:
        """Host copy of the bitset rows, [n, ceil(n/8)] (engine.py:186-188 layout)."""
        return np.ascontiguousarray(self._cur[:, :self.row_bytes].cpu().numpy())

    def register_matrix(self) -> np.ndarray:
        return self.cur

    def ball_members(self, v: int) -> np.ndarray:
        return np.flatnonzero(np.unpackbits(self.cur[v])[:self.n])
