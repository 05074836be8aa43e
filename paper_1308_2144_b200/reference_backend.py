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
        self.cur = torch.zeros((n, p), dtype=torch.uint8, device=dv)
        self.nxt = torch.empty_like(self.cur)
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
            self.cur.data_ptr(), self.est.data_ptr(), self.n, self.params.b,
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
            self.cur.data_ptr(), self.nxt.data_ptr(), prev_bits.data_ptr(),
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
        self.cur, self.nxt = self.nxt, self.cur

    def counters(self) -> CounterArray:
        return CounterArray.from_dense(self.sched.to_original(self.cur).cpu().numpy(),
                                       self.params)

    def register_matrix(self) -> np.ndarray:
        return self.sched.to_original(self.cur).cpu().numpy()
