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
    """engine.py:138-175 backend protocol over hb_seed / hb_union_step."""

    kind = "probabilistic"

    def __init__(self, n: int, params, graph, device=None, schedule: str = "identity"):
        self.params, self.n = params, n
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.stream = torch.cuda.current_stream(self.device)
        p = params.p
        self.sched = build_schedule(graph.offsets, graph.successors, params.b, self.device,
                                    schedule, stream=self.stream)
        dv = self.device
        self._cur = torch.zeros((n, p), dtype=torch.uint8, device=dv)
        self._nxt = torch.empty_like(self._cur)
        words = max((n + 31) // 32, 1)
        self.bits = [torch.zeros(words, dtype=torch.int32, device=dv) for _ in range(2)]
        self.est = torch.zeros(n, dtype=torch.float64, device=dv)
        self.lc = torch.from_numpy(lc_table(p)).to(dv)
        self.alpha_p2, self.lc_cut, _ = estimator_constants(p)
        self.counts = torch.zeros(2, dtype=torch.int64, device=dv)
        self.t = 0

    # -- protocol --------------------------------------------------------------
    def seed(self, weights, est: np.ndarray) -> None:
        w = None
        if weights is not None:
            w = torch.from_numpy(np.asarray(getattr(weights, "values", weights),
                                            dtype=np.int64)).to(self.device)
        perm = self.sched.perm
        _lib.check(_lib.hb().hb_seed(
            self._cur.data_ptr(), self.est.data_ptr(), self.n, self.params.b,
            self.params.register_width, self.params.seed & ((1 << 64) - 1),
            perm.data_ptr() if perm is not None else None,
            w.data_ptr() if w is not None else None, self.lc.data_ptr(), self.alpha_p2,
            self.lc_cut, self.stream.cuda_stream), "hb_seed")
        if self.n:
            est[:] = self.sched.to_original(self.est).cpu().numpy()

    def union_range(self, lo, hi, offsets, successors, changed_prev, changed_now, est,
                    new_est, skip_stable) -> int:
        """One call per iteration over [0, n) (use workers=1 with this backend)."""
        if (lo, hi) != (0, self.n):
            raise ValueError("CudaBackend processes the whole graph per call (workers=1)")
        self.t += 1
        s = self.sched
        prev = torch.from_numpy(np.packbits(np.asarray(changed_prev, dtype=bool),
                                            bitorder="little"))
        prev_dev = torch.zeros_like(self.bits[0]).view(torch.uint8)
        prev_dev[:prev.numel()].copy_(prev.to(self.device))
        prev_bits = s.to_internal_bits(prev_dev.view(torch.int32), self.n)
        self.est.copy_(s.to_internal(torch.from_numpy(np.ascontiguousarray(est)).to(self.device)))
        dense = (not skip_stable) or bool(np.all(changed_prev))
        _lib.check(_lib.hb().hb_union_step(
            self.n, s.light_lo, s.light_hi, s.offsets.data_ptr(), s.succ.data_ptr(),
            self._cur.data_ptr(), self._nxt.data_ptr(), prev_bits.data_ptr(),
            self.bits[1].data_ptr(), 1, self.est.data_ptr(), None, None, self.t,
            self.lc.data_ptr(), self.alpha_p2, self.lc_cut, self.params.b, int(dense),
            s.light_max_deg, s.heavy_nodes.data_ptr(), s.item_first.data_ptr(), s.n_heavy,
            s.finish_order.data_ptr(), s.n_mega, s.item_node.data_ptr(), s.item_beg.data_ptr(),
            s.n_items, s.item_arcs, s.partial.data_ptr(), self.counts.data_ptr(),
            self.counts.data_ptr() + 8, s.hot_rows, None, 0, 0, None, 0, None, 0, None, None,
            self.stream.cuda_stream), "hb_union_step")
        new_est[:] = s.to_original(self.est).cpu().numpy()
        now = s.to_original_bits(self.bits[1], self.n).cpu().numpy()
        changed_now[:] = now
        return int(self.counts[0].item())

    def swap(self) -> None:
        self._cur, self._nxt = self._nxt, self._cur

    @property
    def cur(self) -> np.ndarray:
        """Host copy of the rows in original order (what the reference's
        HyperBallState.register_matrix / save read from backend.cur)."""
        return self.register_matrix()

    def counters(self) -> CounterArray:
        return CounterArray.from_dense(self.register_matrix(), self.params)

    def register_matrix(self) -> np.ndarray:
        return self.sched.to_original(self._cur).cpu().numpy()


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
