"""Batched repeated runs: R seeds in one union pass (cli.py:222-254).

The reference CLI repeats ``engine.run`` with seeds s, s+1, ... and aggregates the
centralities (``multi_run_aggregate``, centrality.py:179-193).  Runs share the graph, so
on the device R of them share one CSR scan: a row of the register array holds the R runs'
registers side by side (R * p bytes; run r at bytes [r*p, (r+1)*p)), the union is the
same byte-wise max over the wide row, and ``hb_union_step_runs`` does the change test,
estimate and accumulate per run.  At small p this is also what HBM wants: a random 16-byte
row costs a 64-byte DRAM burst, four 16-byte runs fill it.

Every run's registers, estimates, iteration count and sums are bit-identical to an
independent run with its seed (tests/test_gpu_multirun.py): the source skip uses the OR
of the runs' change flags, and merging an unchanged source is a no-op.  A converged run
keeps riding along unchanged (its deltas are zero) until every run has converged.

At the end each run gets an ordinary ``HyperBallState``: its registers and estimates are
sliced out of the batch (still in the batch schedule's node order, which serves every
host view), and the single-run schedule is only built if the state is iterated again.
Each run's accumulator stays bound to its device sums, so ``finalize_*`` runs on the
device as after ``run``.
"""

from __future__ import annotations

import ctypes
import time
import weakref
from dataclasses import replace

import numpy as np
import torch

from . import _lib
from .centrality import MAX_FUSED_DISCOUNTS, CentralityAccumulator
from .engine import (DENSE_FRAC, FRONTIER_DIV, ConvergenceError, HyperBallConfig, HyperBallState, _Device,
                     _DeviceSums, _PINNED, _check_weighted_width, _graph_arrays,
                     _resolve_device, _weights_array)
from .hll import estimator_constants, lc_table
from .schedule import build_schedule

MAX_ROW_BYTES = 256    # widest batched row the kernels are built for
MAX_RUNS = 16


def batch_size(p: int, runs: int) -> int:
    """Default runs per batch: fill a 64-byte DRAM burst per row (p = 16 -> 4, p = 32 -> 2),
    never more than `runs`; 1 (no batching) from p = 64 up."""
    if p >= 64 or runs < 2:
        return 1
    return min(runs, 64 // p)


def supported(config: HyperBallConfig, batch: int, discounts=()) -> bool:
    p = config.params.p
    return (batch >= 2 and batch & (batch - 1) == 0 and batch <= MAX_RUNS
            and batch * p <= MAX_ROW_BYTES and config.backend == "probabilistic"
            and len(discounts) <= MAX_FUSED_DISCOUNTS
            and all(hasattr(d, "device_factor") for d in discounts))


class _Batch:
    """Device state of R = 2^k runs sharing one wide-row register array."""

    def __init__(self, g, config: HyperBallConfig, seeds, weights, discounts=()):
        pr = config.params
        self.specs = list(discounts)
        self.R = len(seeds)
        self.log2r = self.R.bit_length() - 1
        self.b, self.p = pr.b, pr.p
        self.device = _resolve_device(config.device)
        self.stream = torch.cuda.current_stream(self.device)
        off, suc = _graph_arrays(g)
        with torch.cuda.device(self.device):
            self.sched = build_schedule(off, suc, self.b + self.log2r, self.device,
                                        config.schedule, 1, 0, self.stream)
        s = self.sched
        n, R, p, dv = s.n, self.R, self.p, self.device
        self.n = n
        words = max((n + 31) // 32, 1)
        self.words = words
        self.cur = torch.empty((n, R * p), dtype=torch.uint8, device=dv)
        self.nxt = torch.empty_like(self.cur)
        self.est = torch.zeros((R, n), dtype=torch.float64, device=dv)
        self.sum_dist = torch.zeros((R, n), dtype=torch.float64, device=dv)
        self.sum_recip = torch.zeros((R, n), dtype=torch.float64, device=dv)
        self.disc = torch.zeros((R, len(self.specs), n), dtype=torch.float64, device=dv)
        self.chg_prev = torch.full((words,), -1, dtype=torch.int32, device=dv)
        self.chg_now = torch.zeros((words,), dtype=torch.int32, device=dv)
        self.chg_runs = torch.zeros((R, words), dtype=torch.int32, device=dv)
        self.counts = torch.zeros(2 + R, dtype=torch.int64, device=dv)  # any, merged, per run
        self.lc = torch.from_numpy(lc_table(p)).to(dv)
        self.alpha_p2, self.lc_cut, _ = estimator_constants(p)
        self.active = None
        self.launches = 0
        L = _lib.hb()
        w = None if weights is None else torch.from_numpy(
            np.ascontiguousarray(weights, dtype=np.int64)).to(dv)
        tmp = torch.empty((n, p), dtype=torch.uint8, device=dv)
        view = self.cur.view(n, R, p)
        perm = s.perm
        for r, seed in enumerate(seeds):
            _lib.check(L.hb_seed(tmp.data_ptr(), self.est[r].data_ptr(), n, self.b,
                                 pr.register_width, seed & ((1 << 64) - 1),
                                 perm.data_ptr() if perm is not None else None,
                                 w.data_ptr() if w is not None else None, self.lc.data_ptr(),
                                 self.alpha_p2, self.lc_cut, self.stream.cuda_stream), "hb_seed")
            with torch.cuda.stream(self.stream):
                view[:, r].copy_(tmp)
            self.launches += 1 if n else 0
        del tmp
        self.full_pass = True
        if s.light_hi_steady < s.light_hi:        # zero in-degree suffix: see _Device.seed
            with torch.cuda.stream(self.stream):
                self.nxt.copy_(self.cur)
            self.full_pass = False
        self.prev_all = True
        self.last_nch = None

    def _frontier(self, dense: bool):
        s = self.sched
        if dense or self.last_nch is None or self.last_nch * FRONTIER_DIV >= self.n:
            return None
        if self.active is None:
            self.active = torch.empty_like(self.chg_now)
        _lib.check(_lib.hb().hb_mark_pull(
            self.n, s.offsets.data_ptr(), s.succ.data_ptr(), self.chg_prev.data_ptr(),
            self.active.data_ptr(), s.light_max_deg, s.item_node.data_ptr(),
            s.item_beg.data_ptr(), s.n_items, s.item_arcs, self.stream.cuda_stream),
            "hb_mark_pull")
        self.launches += 1 + (1 if s.n_items else 0)
        return self.active.data_ptr()

    def step(self, t: int, dense: bool, frontier: bool):
        """One batched iteration; returns (changed nodes (any run), per-run changed list)."""
        s = self.sched
        active = self._frontier(dense) if frontier else None
        light_hi = s.light_hi if self.full_pass else s.light_hi_steady
        c = self.counts
        k = len(self.specs)
        scale = (ctypes.c_double * max(k, 1))()
        div = 0
        for i, spec in enumerate(self.specs):
            dflag, f = spec.device_factor(t)
            scale[i] = f
            div |= int(dflag) << i
        _lib.check(_lib.hb().hb_union_step_runs(
            self.n, s.light_lo, light_hi, s.offsets.data_ptr(), s.succ.data_ptr(),
            self.cur.data_ptr(), self.nxt.data_ptr(), self.chg_prev.data_ptr(),
            self.chg_now.data_ptr(), self.chg_runs.data_ptr(), self.est.data_ptr(),
            self.sum_dist.data_ptr(), self.sum_recip.data_ptr(), self.n, t,
            self.lc.data_ptr(), self.alpha_p2, self.lc_cut, self.b, self.log2r, int(dense),
            s.light_max_deg, s.heavy_nodes.data_ptr(), s.item_first.data_ptr(), s.n_heavy,
            s.finish_order.data_ptr(), s.n_mega, s.item_node.data_ptr(), s.item_beg.data_ptr(),
            s.n_items, s.item_arcs, s.partial.data_ptr(), c.data_ptr(), c.data_ptr() + 8,
            c.data_ptr() + 16, s.hot_rows, self.disc.data_ptr() if k else None, self.n, k,
            ctypes.cast(scale, ctypes.c_void_p) if k else None, div, active,
            self.stream.cuda_stream),
            "hb_union_step_runs")
        self.launches += ((light_hi > s.light_lo) + (s.n_items > 0) + (s.n_heavy > 0)
                          + (s.n_mega > 0 and s.n_heavy > s.n_mega) + 1)
        host = c.cpu().tolist()
        self.last_nch = host[0]
        self.cur, self.nxt = self.nxt, self.cur
        self.chg_prev, self.chg_now = self.chg_now, self.chg_prev
        self.prev_all = False
        self.full_pass = False
        return host[0], host[2:]

    def host_est(self, r: int, src=None) -> np.ndarray:
        x = self.est[r] if src is None else src[r]
        return _to_host(self.sched.to_original(x), self.stream)


def _to_host(x: torch.Tensor, stream) -> np.ndarray:
    arr, tv = _PINNED.array(tuple(x.shape), x.dtype)
    tv.copy_(x, non_blocking=True)
    stream.synchronize()
    return arr.copy()


def run_batched(g, config: HyperBallConfig, seeds, observers, discounts=()):
    """Runs with `seeds` (len a power of two, <= 16, len * p <= 256) in one batch.
    observers[r]: run r's observers (a CentralityAccumulator among them, with `discounts`,
    is folded on the device).  Progress lines (config.progress) are written run after run
    once the batch is done, in the reference's format.  Returns the per-run states."""
    n = (g.offsets.numel() if isinstance(g.offsets, torch.Tensor)
         else np.asarray(g.offsets).shape[0]) - 1
    w = _weights_array(config.weights, n)
    if w is not None:
        _check_weighted_width(config.params, w)
    R = len(seeds)
    cfgs = [replace(config, params=replace(config.params, seed=sd)) for sd in seeds]
    if n == 0:
        from .engine import run
        return [run(g, c, obs) for c, obs in zip(cfgs, observers)]
    bt = _Batch(g, config, seeds, w, discounts)
    names = [d.name for d in discounts]
    fused = [next((o for o in obs if isinstance(o, CentralityAccumulator) and o.n == n
                   and [d.name for d in o.discounts] == names), None) for obs in observers]
    lines = [[] for _ in range(R)]
    generic = [[o for o in obs if o is not f] for obs, f in zip(observers, fused)]
    need_old = any(generic)
    done = [False] * R
    t_run = [0] * R

    def _finish(r):
        # hand run r an ordinary single-run state: its device arrays are sliced out of the
        # batch (internal order of the batch schedule); the single-run schedule is only
        # built if the state is iterated again (graph_key None -> _Device.bind_graph)
        view = bt.cur.view(n, R, bt.p)          # bt.cur: the buffer of the latest step
        dev = _parked_device(bt, cfgs[r], view[:, r].contiguous(), bt.est[r].clone())
        st = HyperBallState(cfgs[r], n, dev)
        st.t, st.num_changed = t_run[r], 0
        if fused[r] is not None:
            _bind_batch_sums(st, fused[r], bt.sum_dist[r], bt.sum_recip[r], bt.disc[r],
                             bt.specs)
        final = st.est
        final.setflags(write=False)
        for obs in observers[r]:
            obs.on_converged(final)
        return st

    t = 0
    while True:
        t += 1
        started = time.perf_counter()
        dense = (bt.prev_all or not config.skip_stable_nodes
                 or (bt.last_nch is not None and bt.last_nch >= DENSE_FRAC * n))
        old = bt.est.clone() if need_old else None
        _, per_run = bt.step(t, dense, config.frontier)
        elapsed_ms = (time.perf_counter() - started) * 1000.0
        for r in range(R):
            if done[r]:
                continue
            if config.progress is not None:
                lines[r].append(f"t={t} changed={per_run[r]} elapsed_ms={elapsed_ms:.0f}\n")
            if generic[r]:
                o_h, n_h = bt.host_est(r, old), bt.host_est(r)
                o_h.setflags(write=False)
                n_h.setflags(write=False)
                for obs in generic[r]:
                    obs.on_step(t, o_h, n_h)
            if per_run[r] == 0:
                done[r], t_run[r] = True, t
            elif config.max_iterations is not None and t >= config.max_iterations:
                # The reference runs the seeds one after another (cli.py:222-254): every
                # earlier run has converged (a non-converged earlier run would have raised
                # first, at a lower r), written its progress lines and received
                # on_converged before run r raises; later runs never start.
                if config.progress is not None:
                    for q in range(r + 1):
                        config.progress.write("".join(lines[q]))
                for q in range(r):
                    _finish(q)
                raise ConvergenceError(t, per_run[r])
        if all(done):
            break
    if config.progress is not None:
        for r in range(R):
            config.progress.write("".join(lines[r]))
    return [_finish(r) for r in range(R)]


def _parked_device(bt: _Batch, cfg: HyperBallConfig, cur: torch.Tensor,
                   est: torch.Tensor) -> _Device:
    """A converged single-run _Device over the batch schedule (order conversions only)."""
    dev = object.__new__(_Device)
    n = bt.n
    dev.params, dev.b, dev.p = cfg.params, bt.b, bt.p
    dev.device, dev.stream = bt.device, bt.stream
    dev.order = bt.sched.order
    dev.world, dev.rank_id = 1, 0
    dev.sched, dev.n, dev.graph_key = bt.sched, n, None
    dev.cur, dev.nxt = cur, cur.clone()
    dev.chg_prev = torch.zeros_like(bt.chg_prev)
    dev.chg_now = torch.zeros_like(bt.chg_now)
    dev.est = est
    dev.lc, dev.alpha_p2, dev.lc_cut = bt.lc, bt.alpha_p2, bt.lc_cut
    dev.counts = torch.zeros(2, dtype=torch.int64, device=bt.device)
    dev.ticket = torch.zeros(1, dtype=torch.int64, device=bt.device)
    dev.merged_total = 0
    dev.prev_all = dev.full_pass = False
    dev.launches = dev.launches_at_last_step = bt.launches
    dev.frontier = cfg.frontier
    dev.fwd = dev.active = dev.last_nch = None
    dev._sparse_run = 0
    dev._seed_weights = None
    return dev


def _bind_batch_sums(st: HyperBallState, acc, sum_dist: torch.Tensor,
                     sum_recip: torch.Tensor, disc: torch.Tensor, specs) -> None:
    """Leave run r's sums on the device as the accumulator's binding (device finalize);
    reference accumulators (foreign classes) get host copies."""
    dev = st._dev
    if not isinstance(acc, CentralityAccumulator):
        acc.sum_dist = _to_host(dev.sched.to_original(sum_dist), dev.stream)
        acc.sum_recip = _to_host(dev.sched.to_original(sum_recip), dev.stream)
        return
    sums = object.__new__(_DeviceSums)
    sums.dev = dev
    sums._acc = weakref.ref(acc)
    sums.foreign = False
    sums.host_ids = (id(acc._sum_dist), id(acc._sum_recip))
    sums.specs = list(specs)
    sums.sum_dist, sums.sum_recip = sum_dist, sum_recip
    sums.disc = disc
    sums.dirty, sums.stale = True, False
    acc._binding = sums
    acc._fresh = False
    st._sums = sums
