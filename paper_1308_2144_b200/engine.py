"""Ball-growth engine on the B200: the reference's public API (engine.py:52-435) over
device-resident state and the sm_100a kernels of ``libhyperball_b200.so``.

Drop-in surface (same names, argument meanings, errors and result layout as
/root/reference/pkg/src/hyperball/engine.py):

* ``HyperBallConfig``  engine.py:82-97, plus ``device`` and ``schedule`` (B200 fields)
* ``HyperBallState``   engine.py:216-280 (``t``, ``num_changed``, ``est``,
  ``changed_prev``, ``estimates()``, ``register_matrix()``, ``counters()``, ``save``)
* ``initialize`` / ``iterate`` / ``run`` / ``resume`` / ``load_state``
  engine.py:283-435, ``ConvergenceError`` engine.py:52-60, ``BallObserver`` 63-79.

What runs where: the graph (CSR of G^T), both register buffers, the change bitmaps, the
estimates and the fused accumulator sums live in HBM for the whole run.  One iteration is
one ``hb_union_step`` call (heavy-item pass, light pass, heavy finish) plus a
single 8-byte read-back of the changed count, which is the loop's termination test
exactly as in engine.py:390,426-427.  Host copies are made only when a caller asks for
them (``state.est``, ``register_matrix()``, a non-fused observer).  There is no CPU
fallback: without a CUDA device or the built library every entry point raises.
"""

from __future__ import annotations

import ctypes
import io
import math
import weakref
import struct
import time
from dataclasses import dataclass, field
from typing import IO, Iterable

import numpy as np
import torch

from . import _lib
from .centrality import BallObserver, CentralityAccumulator, fusable
from .hll import CounterArray, CounterParams, estimator_constants, lc_table
from .schedule import Schedule, build_schedule, die_eligible, pack_bits, unpack_bits

import os as _os

# frontier mode when fewer than n / FRONTIER_DIV counters changed in the last iteration
FRONTIER_DIV = int(_os.environ.get("HB_FRONTIER_DIV", "8"))
# ... marked by one streaming pass over G^T's ids (hb_mark_pull) up to the FRONTIER_AFTER-th
# consecutive such iteration, from the forward graph (hb_mark_active) after it (building
# the forward graph costs several full scans; short tails do not repay it)
FRONTIER_AFTER = int(_os.environ.get("HB_FRONTIER_AFTER", "4"))

# a step runs dense (no per-source change test) when at least this fraction of the counters
# changed in the previous iteration
DENSE_FRAC = float(_os.environ.get("HB_DENSE_FRAC", "0.95"))
# ... or when the counters that changed are the sources of at least DENSE_ARC_FRAC of the
# arcs (estimated on the device from FLAG_SAMPLES random arcs, hb_sample_flagged_arcs;
# graphs of FLAG_MIN_ARCS arcs and more): on R-MAT a third of the nodes change but they
# feed 99% of the arcs, and the per-source test then costs more than the merges it saves.
DENSE_ARC_FRAC = float(_os.environ.get("HB_DENSE_ARC_FRAC", "0.7"))
FLAG_MIN_ARCS = 1 << 26
FLAG_SAMPLES = 1 << 16
# pull marking with a shared-memory filter of the changed nodes at or below this many
FILTER_MAX_CHANGED = int(_os.environ.get("HB_FILTER_MAX_CHANGED", "8192"))

CHECKPOINT_MAGIC = b"HBCK"
CHECKPOINT_VERSION = 1

BACKEND_PROBABILISTIC = "probabilistic"
BACKEND_EXACT = "exact"
# "cuda": the name a reference-side registration would use for this engine
_BACKEND_ALIASES = {"hll": BACKEND_PROBABILISTIC, "cuda": BACKEND_PROBABILISTIC}


class ConvergenceError(RuntimeError):
    """Safety-cap overrun; reports the iteration and open counter count."""

    def __init__(self, t: int, num_changed: int):
        super().__init__(f"max_iterations reached at t={t} with {num_changed} counters "
                         f"still changing")
        self.t = t
        self.num_changed = num_changed


@dataclass
class HyperBallConfig:
    params: CounterParams = field(default_factory=lambda: CounterParams(b=6))
    weights: object | None = None
    backend: str = BACKEND_PROBABILISTIC
    workers: int = 1
    max_iterations: int | None = None
    skip_stable_nodes: bool = True
    progress: IO[str] | None = None
    device: object | None = None        # B200: CUDA device (index, "cuda:k" or None = current)
    schedule: str = "auto"              # B200: "auto" | "identity" | "degree" (schedule.py)
    frontier: bool = True               # B200: sparse iterations visit only the frontier

    def __post_init__(self) -> None:
        self.backend = _BACKEND_ALIASES.get(self.backend, self.backend)
        if self.backend not in (BACKEND_PROBABILISTIC, BACKEND_EXACT):
            raise ValueError(f"unknown counter backend {self.backend!r}")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.schedule not in ("auto", "identity", "degree", "window"):
            raise ValueError(f"unknown schedule {self.schedule!r}")


# ---------------------------------------------------------------------------- helpers

def _weights_array(weights, n: int):
    if weights is None:
        return None
    vals = np.asarray(getattr(weights, "values", weights), dtype=np.int64)
    if vals.shape[0] != n:
        raise ValueError(f"weights length {vals.shape[0]} != node count {n}")
    if n and vals.min() < 1:
        raise ValueError("node weights must be >= 1")
    return vals


def _check_weighted_width(params: CounterParams, vals: np.ndarray) -> None:
    """Registers must be able to reach log2(total weight) (engine.py:122-135)."""
    total = max(int(vals.sum()), 2)
    needed = math.log2(total)
    if params.saturation < math.ceil(needed):
        raise ValueError(
            f"register_width={params.register_width} saturates at {params.saturation}, "
            f"below log2(total weight) = {needed:.1f}; register_width 6 (or wider) is "
            f"required for this weighting")


def _resolve_device(dev) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1308_2144_b200 needs a CUDA device (no CPU fallback)")
    if dev is None:
        return torch.device("cuda", torch.cuda.current_device())
    if isinstance(dev, int):
        return torch.device("cuda", dev)
    d = torch.device(dev)
    if d.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {dev!r}")
    return d if d.index is not None else torch.device("cuda", torch.cuda.current_device())


class _PinnedPool:
    """Page-locked host blocks for device->host copies, recycled when the numpy array
    handed to the caller is garbage-collected (page-locking 100+ MB costs tens of ms, a
    recycled block costs nothing; the copy itself then runs at full PCIe rate)."""

    def __init__(self):
        import threading
        self._free: dict = {}
        self._lock = threading.Lock()

    def array(self, shape, dtype: torch.dtype):
        """(numpy array, the pinned torch tensor viewing the same memory)."""
        import weakref
        numel = int(np.prod(shape)) if len(shape) else 1
        key = (numel, dtype)
        with self._lock:
            lst = self._free.get(key)
            t = lst.pop() if lst else None
        if t is None:
            t = torch.empty(numel, dtype=dtype, pin_memory=True)
        tv = t.view(shape)
        arr = tv.numpy()
        weakref.finalize(arr, self._give_back, key, t)
        return arr, tv

    def _give_back(self, key, t) -> None:
        with self._lock:
            self._free.setdefault(key, []).append(t)


_PINNED = _PinnedPool()


def _graph_arrays(g):
    return g.offsets, g.successors


def _graph_key(g):
    off, suc = _graph_arrays(g)
    return (id(off), id(suc), int(np.asarray(off).shape[0]) - 1 if not isinstance(off, torch.Tensor)
            else off.numel() - 1)


class _DeviceSums:
    """Device-resident CentralityAccumulator sums (internal node order)."""

    @property
    def acc(self):
        return self._acc()

    def __init__(self, dev: "_Device", acc):
        self.dev = dev
        self._acc = weakref.ref(acc)   # no acc <-> binding cycle: results free promptly
        self.foreign = not isinstance(acc, CentralityAccumulator)
        if self.foreign:
            sd, sr = acc.sum_dist, acc.sum_recip
        else:
            sd, sr = acc._sum_dist, acc._sum_recip
        self.host_ids = (id(sd), id(sr))
        self.specs = [] if self.foreign else list(acc.discounts)
        k = len(self.specs)
        if not self.foreign and acc._fresh:       # nothing accumulated yet: no upload
            self.sum_dist = torch.zeros(dev.n, dtype=torch.float64, device=dev.device)
            self.sum_recip = torch.zeros(dev.n, dtype=torch.float64, device=dev.device)
            self.disc = torch.zeros((k, dev.n), dtype=torch.float64, device=dev.device)
        else:
            self.sum_dist = dev.to_internal(np.asarray(sd, dtype=np.float64))
            self.sum_recip = dev.to_internal(np.asarray(sr, dtype=np.float64))
            self.disc = torch.zeros((k, dev.n), dtype=torch.float64, device=dev.device)
            for i, spec in enumerate(self.specs):
                self.disc[i] = dev.to_internal(np.asarray(acc._discounted[spec.name],
                                                          dtype=np.float64))
        self.dirty = False
        self.stale = False

    def disc_args(self, t: int):
        """(base ptr, stride, count, host scale array, divide mask) for hb_union_step."""
        import ctypes
        k = len(self.specs)
        if k == 0:
            return None, 0, 0, None, 0
        scale = (ctypes.c_double * k)()
        div = 0
        for i, spec in enumerate(self.specs):
            d, f = spec.device_factor(t)
            scale[i] = f
            div |= int(d) << i
        self._scale_keepalive = scale
        return self.disc.data_ptr(), self.dev.n, k, ctypes.cast(scale, ctypes.c_void_p), div

    coreach_dev = None
    coreach_version = None

    def capture_coreach(self, version) -> None:
        """on_converged: keep the final estimates on the device for finalize_lin, tagged
        with the accumulator's coreach version (a later reassignment invalidates it)."""
        self.coreach_dev = self.dev.est.clone()
        self.coreach_version = version

    def fetch_coreach(self) -> np.ndarray:
        """Host copy (original order, read-only) of the captured final estimates."""
        out = self.dev.to_host(self.coreach_dev)
        out.setflags(write=False)
        return out

    _fin_cache = None   # (key, {name: host array}, {name: handed out once})

    def finalize(self, which: str) -> np.ndarray:
        """closeness / harmonic / lin on the device, in original order, each computed
        (hb_finalize with that output only) and copied to the host on its first request:
        a harmonic-only caller reads one sum array and downloads n doubles, not 3n."""
        dev = self.dev
        key = (dev.launches_at_last_step, self.coreach_version)
        if self._fin_cache is None or self._fin_cache[0] != key:
            self._fin_cache = (key, {}, {})
        _, device_rows, host = self._fin_cache
        if which == "lin" and self.coreach_dev is None:
            return None
        if which not in device_rows:
            n = dev.n
            out = torch.empty(n, dtype=torch.float64, device=dev.device)
            rank = dev.sched.rank
            ptr = {nm: (out.data_ptr() if nm == which else None)
                   for nm in ("closeness", "harmonic", "lin")}
            _lib.check(_lib.hb().hb_finalize(
                n, rank.data_ptr() if rank is not None else None, self.sum_dist.data_ptr(),
                self.sum_recip.data_ptr(),
                self.coreach_dev.data_ptr() if which == "lin" else None, ptr["closeness"],
                ptr["harmonic"], ptr["lin"], dev.stream.cuda_stream), "hb_finalize")
            dev.launches += 1
            device_rows[which] = out
        if which in host:                  # the reference returns a fresh array per call
            return host[which].copy()
        host[which] = dev.to_host_raw(device_rows[which])
        return host[which]

    def pull_into(self, acc) -> None:
        sd = self.dev.to_host(self.sum_dist)
        sr = self.dev.to_host(self.sum_recip)
        self.dirty = False
        if self.foreign:
            acc.sum_dist, acc.sum_recip = sd, sr
            self.host_ids = (id(acc.sum_dist), id(acc.sum_recip))
        else:
            acc._sum_dist, acc._sum_recip = sd, sr
            acc._discounted = {spec.name: self.dev.to_host(self.disc[i])
                               for i, spec in enumerate(self.specs)}
            acc._fresh = False

    def invalidate(self) -> None:
        self.stale = True

    def reorder(self, old, new) -> None:
        """The device state moved to schedule `new`: reorder the sums from `old`."""
        def mv(x):
            return new.to_internal(old.to_original(x)).contiguous()
        self.sum_dist, self.sum_recip = mv(self.sum_dist), mv(self.sum_recip)
        if self.disc.numel():
            self.disc = torch.stack([mv(row) for row in self.disc])
        if self.coreach_dev is not None:
            self.coreach_dev = mv(self.coreach_dev)
        self._fin_cache = None

    def still_valid(self) -> bool:
        if self.stale:
            return False
        if self.foreign:
            return self.host_ids == (id(self.acc.sum_dist), id(self.acc.sum_recip))
        return True


class _Device:
    """Per-run device resources; all per-node arrays are in internal (schedule) order."""

    def __init__(self, g, config: HyperBallConfig, world: int = 1, rank_id: int = 0,
                 seed_weights=False):
        """seed_weights: False = do not seed; None or an int64 array = seed (as seed())
        while the successor ids are still being uploaded (build_schedule's on_order)."""
        self.params = config.params
        self.b = config.params.b
        self.p = config.params.p
        L = _lib.hb()
        if not (L.hb_min_log2m() <= self.b <= L.hb_max_log2m()):
            raise ValueError(f"log2m b={self.b} outside the built range "
                             f"[{L.hb_min_log2m()}, {L.hb_max_log2m()}]")
        self.device = _resolve_device(config.device)
        self.stream = torch.cuda.current_stream(self.device)
        self.order = config.schedule
        self.world, self.rank_id = world, rank_id
        off, _ = _graph_arrays(g)
        n = (off.numel() if isinstance(off, torch.Tensor) else np.asarray(off).shape[0]) - 1
        p = self.p
        words = max((n + 31) // 32, 1)
        dv = self.device
        self.cur = torch.empty((n, p), dtype=torch.uint8, device=dv)
        self.nxt = torch.empty((n, p), dtype=torch.uint8, device=dv)
        self.chg_prev = torch.full((words,), -1, dtype=torch.int32, device=dv)
        self.chg_now = torch.zeros((words,), dtype=torch.int32, device=dv)
        self.est = torch.zeros(n, dtype=torch.float64, device=dv)
        self.lc = torch.from_numpy(lc_table(p)).to(dv)
        self.alpha_p2, self.lc_cut, _ = estimator_constants(p)
        self.counts = torch.zeros(2, dtype=torch.int64, device=dv)   # [changed, merged arcs]
        self.ticket = torch.zeros(2, dtype=torch.int64, device=dv)   # chunk / item tickets
        self.merged_total = 0         # arcs whose source row was merged, all iterations
        self.prev_all = True          # chg_prev is all-ones (first iteration)
        self.full_pass = True         # zero in-degree nodes may still need their copy
        self.launches = 0             # kernels launched by hb_union_step calls
        self.launches_at_last_step = 0
        self.frontier = config.frontier
        self.fwd = None               # forward CSR (internal ids), built on first use
        self.active = None
        self.last_nch = None
        self.slice_counts = None      # per-slice counters of a streamed iteration 1
        self.flag_out = None          # device: arcs whose source changed (last step)
        self.change_filter = None     # device: hash filter of the changed nodes
        self.last_flagged = None
        early = None
        if seed_weights is not False:
            def early(perm):
                self._launch_seed(seed_weights, perm)
        self._build_graph(g, on_order=early)
        if self.sched.local:
            self.frontier = False        # frontier marking scans every row's ids
        if early is not None:
            self._after_seed()

    def fresh(self, config: HyperBallConfig) -> "_Device":
        """A new device state for another run on the same graph and schedule."""
        other = object.__new__(type(self))
        other.__dict__.update(self.__dict__)
        other.params = config.params
        n, p = self.n, self.p
        dv = self.device
        other.cur = torch.empty((n, p), dtype=torch.uint8, device=dv)
        other.nxt = torch.empty((n, p), dtype=torch.uint8, device=dv)
        other.chg_prev = torch.full_like(self.chg_prev, -1)
        other.chg_now = torch.zeros_like(self.chg_now)
        other.est = torch.zeros(n, dtype=torch.float64, device=dv)
        other.counts = torch.zeros(2, dtype=torch.int64, device=dv)
        other.ticket = torch.zeros(2, dtype=torch.int64, device=dv)
        other.merged_total = 0
        other.prev_all = True
        other.full_pass = True
        other.launches = 0
        other.launches_at_last_step = 0
        other.active = None
        other.last_nch = None
        other.slice_counts = None
        other.flag_out = None
        other.last_flagged = None
        other._sparse_run = 0
        return other

    # -- graph ---------------------------------------------------------------
    def _build_graph(self, g, on_order=None) -> None:
        off, suc = _graph_arrays(g)
        with torch.cuda.device(self.device):
            self.sched: Schedule = build_schedule(off, suc, self.b, self.device, self.order,
                                                  self.world, self.rank_id, self.stream,
                                                  on_order=on_order)
        self.n = self.sched.n
        self.graph_key = _graph_key(g)

    def bind_graph(self, g):
        """Schedule `g` (a no-op for the graph already bound).  Returns the previous
        Schedule when it was replaced (per-node device arrays kept elsewhere, e.g. the
        accumulator sums, must then be reordered), else None."""
        if _graph_key(g) == self.graph_key:
            return None
        off, _ = _graph_arrays(g)
        n_new = (off.numel() if isinstance(off, torch.Tensor) else np.asarray(off).shape[0]) - 1
        if n_new != self.n:
            raise ValueError(f"graph has {n_new} nodes, state has {self.n}")
        # different graph object: carry the state over in original order
        snap = self.snapshot_original()
        old = self.sched
        self._build_graph(g)
        self.restore_original(*snap)
        return old

    # -- order conversion ----------------------------------------------------
    def to_internal(self, host_or_dev) -> torch.Tensor:
        x = host_or_dev
        if not isinstance(x, torch.Tensor):
            x = torch.from_numpy(np.ascontiguousarray(x))
        return self.sched.to_internal(x.to(self.device)).contiguous()

    def to_host(self, x: torch.Tensor) -> np.ndarray:
        """Original-order host copy (through pinned memory: full PCIe rate)."""
        return self.to_host_raw(self.sched.to_original(x))

    def to_host_raw(self, x: torch.Tensor) -> np.ndarray:
        arr, tv = _PINNED.array(tuple(x.shape), x.dtype)
        tv.copy_(x, non_blocking=True)
        self.stream.synchronize()
        return arr

    def snapshot_original(self):
        s = self.sched
        cur = s.to_original(self.cur)
        nxt = s.to_original(self.nxt)
        est = s.to_original(self.est)
        prev = s.to_original(unpack_bits(self.chg_prev, self.n))
        return cur, nxt, est, prev

    def restore_original(self, cur, nxt, est, prev) -> None:
        s = self.sched
        self.cur = s.to_internal(cur).contiguous()
        self.nxt = s.to_internal(nxt).contiguous()
        self.est = s.to_internal(est).contiguous()
        self.chg_prev = pack_bits(s.to_internal(prev))

    # -- kernels -------------------------------------------------------------
    def seed(self, weights: np.ndarray | None) -> None:
        self._launch_seed(weights, self.sched.perm)
        self._after_seed()

    def _launch_seed(self, weights, perm) -> None:
        w = None
        if weights is not None:
            w = torch.from_numpy(np.ascontiguousarray(weights, dtype=np.int64)).to(self.device)
        _lib.check(_lib.hb().hb_seed(
            self.cur.data_ptr(), self.est.data_ptr(), self.cur.shape[0], self.b,
            self.params.register_width, self.params.seed & ((1 << 64) - 1),
            perm.data_ptr() if perm is not None else None,
            w.data_ptr() if w is not None else None, self.lc.data_ptr(), self.alpha_p2,
            self.lc_cut, self.stream.cuda_stream), "hb_seed")
        self.launches += 1 if self.cur.shape[0] else 0
        self._seed_weights = w

    def _after_seed(self) -> None:
        s = self.sched
        if s.light_hi_steady < s.light_hi or self.world > 1:
            # Degree order: the zero in-degree suffix never changes, so seed its rows into
            # both buffers (one copy per run) and let iteration 1 skip those nodes too --
            # on R-MAT about half of all nodes (config 5: ~1.7 ms per dense iteration).
            # With several ranks every replica copies all n rows whatever its own slice
            # looks like: a peer's skipped suffix is never pushed, and dense steps read
            # every source row.
            with torch.cuda.stream(self.stream):
                self.nxt.copy_(self.cur)
            if s.light_hi_steady < s.light_hi:
                self.full_pass = False

    def _forward(self):
        """Forward CSR (out-neighbours, internal ids, rows unordered) for frontier marking;
        built once by counting sort (hb_forward_csr)."""
        if self.fwd is None:
            import ctypes
            s, L, st = self.sched, _lib.hb(), self.stream.cuda_stream
            m = s.succ.numel()
            off = torch.empty(self.n + 1, dtype=torch.int64, device=self.device)
            cursor = torch.empty(max(self.n, 1), dtype=torch.int64, device=self.device)
            dst = torch.empty(max(m, 1), dtype=torch.int32, device=self.device)
            tb = ctypes.c_uint64(0)
            _lib.check(L.hb_forward_csr(self.n, s.offsets.data_ptr(), s.succ.data_ptr(), m,
                                        off.data_ptr(), cursor.data_ptr(), dst.data_ptr(),
                                        None, ctypes.byref(tb), st), "hb_forward_csr(size)")
            temp = torch.empty(max(int(tb.value), 1), dtype=torch.uint8, device=self.device)
            _lib.check(L.hb_forward_csr(self.n, s.offsets.data_ptr(), s.succ.data_ptr(), m,
                                        off.data_ptr(), cursor.data_ptr(), dst.data_ptr(),
                                        temp.data_ptr(), ctypes.byref(tb), st),
                       "hb_forward_csr")
            del cursor, temp
            self.fwd = (off, dst)
            self.launches += 2
        return self.fwd

    def _frontier_ptr(self, dense: bool):
        """Device bitmap of the nodes a sparse iteration can touch, or None (full scan).
        Used when fewer than 1/FRONTIER_DIV of the nodes changed last iteration."""
        sparse = (not dense and self.frontier and self.last_nch is not None and self.n > 0
                  and self.last_nch * FRONTIER_DIV < self.n)
        self._sparse_run = getattr(self, "_sparse_run", 0) + 1 if sparse else 0
        if not sparse:
            return None
        if self.active is None:
            self.active = torch.empty_like(self.chg_now)
        s = self.sched
        # the forward graph costs about one atomic per arc (several full scans of the
        # successor lists) to build: only for long sparse tails, or once it exists;
        # before that, one streaming pass over the CSR of G^T marks the frontier
        if self.fwd is None and self._sparse_run < FRONTIER_AFTER:
            L = _lib.hb()
            args = (self.n, s.offsets.data_ptr(), s.succ.data_ptr(), self.chg_prev.data_ptr(),
                    self.active.data_ptr(), s.light_max_deg, s.item_node.data_ptr(),
                    s.item_beg.data_ptr(), s.n_items, s.item_arcs)
            # degree order: the heavy rows are one range, streamed flat; nearly converged:
            # the streamed ids are tested against a shared-memory hash filter of the few
            # changed nodes (hb_mark_pull_filtered)
            h0, h1 = (s.light_lo - s.n_heavy, s.light_lo) if s.order == "degree" else (0, 0)
            filt = None
            if self.last_nch <= FILTER_MAX_CHANGED:
                if self.change_filter is None:
                    self.change_filter = torch.empty(int(L.hb_change_filter_words()),
                                                     dtype=torch.int32, device=self.device)
                filt = self.change_filter.data_ptr()
                self.launches += 1
            _lib.check(L.hb_mark_pull_filtered(*args, h0, h1, filt, self.stream.cuda_stream),
                       "hb_mark_pull_filtered")
            self.launches += 1 if s.n_items else 0
        else:
            off, dst = self._forward()
            _lib.check(_lib.hb().hb_mark_active(self.n, off.data_ptr(), dst.data_ptr(),
                                                self.chg_prev.data_ptr(),
                                                self.active.data_ptr(),
                                                self.stream.cuda_stream), "hb_mark_active")
        self.launches += 1
        return self.active.data_ptr()

    def union_step(self, t: int, dense: bool, sums: _DeviceSums | None, peers=None,
                   clear_chg_now: bool = True, flag_arcs: bool = False) -> int:
        """One hb_union_step.  peers: (n, host uint8** array, host uint32** array[, packed
        row stride]) of peer nxt (or, packed, inbox) / chg_now device addresses for the
        fused multi-GPU push (distributed.py)."""
        s = self.sched
        active = self._frontier_ptr(dense) if peers is None else None
        n_peers, peer_nxt, peer_chg = peers[:3] if peers is not None else (0, None, None)
        pstride = peers[3] if peers is not None and len(peers) > 3 else 0
        light_hi = s.light_hi if self.full_pass else s.light_hi_steady
        sd = sums.sum_dist.data_ptr() if sums is not None else None
        sr = sums.sum_recip.data_ptr() if sums is not None else None
        dargs = sums.disc_args(t) if hasattr(sums, "disc_args") else (None, 0, 0, None, 0)
        # Streamed upload (schedule.py): while successor-id slices are still arriving, the
        # step runs slice by slice, each one as soon as its ids are uploaded (and relabelled)
        # -- the light kernel over that row range, its own counters -- so iteration 1
        # overlaps the rest of the PCIe copy.  Rows are independent within a step.
        parts = [(s.light_lo, light_hi, None)]
        if (s.pending and s.n_items == 0 and n_peers == 0 and active is None
                and s.light_lo == 0 and light_hi == self.n):
            parts = s.take_pending()
        elif s.pending:
            s.ensure_ready()
        if len(parts) > 1 and (self.slice_counts is None
                               or self.slice_counts.shape[0] < len(parts)):
            self.slice_counts = torch.zeros((len(parts), 2), dtype=torch.int64,
                                            device=self.device)
        L = _lib.hb()
        die = self.die_args() if active is None and n_peers == 0 else {}
        for k, (lo, hi, ev) in enumerate(parts):
            if ev is not None:
                s.ready_slice(lo, hi, ev)
            cnt = self.counts if len(parts) == 1 else self.slice_counts[k]
            disc, disc_stride, n_disc, disc_scale, disc_div = dargs
            _lib.union_step(_lib.StepArgs(
                n=self.n, lo=lo, hi=hi, offsets=s.offsets_ptr(),
                succ=s.succ_buf.data_ptr(), cur=self.cur.data_ptr(), nxt=self.nxt.data_ptr(),
                chg_prev=self.chg_prev.data_ptr(), chg_now=self.chg_now.data_ptr(),
                est=self.est.data_ptr(), b=self.b, dense=int(dense),
                clear_chg_now=int(clear_chg_now and k == 0), n_disc=n_disc, t=t,
                lc_table=self.lc.data_ptr(), alpha_p2=self.alpha_p2, lc_cut=self.lc_cut,
                sum_dist=sd, sum_recip=sr, disc=disc, disc_stride=disc_stride,
                disc_scale=disc_scale, disc_div=disc_div, n_peers=n_peers,
                nch_out=cnt.data_ptr(), merged_out=cnt.data_ptr() + 8, active=active,
                peer_nxt=ctypes.cast(peer_nxt, ctypes.c_void_p) if peer_nxt is not None
                else None,
                peer_chg=ctypes.cast(peer_chg, ctypes.c_void_p) if peer_chg is not None
                else None, peer_packed_stride=pstride, ticket=self.ticket.data_ptr(),
                stream=self.stream.cuda_stream, **die, **_lib.schedule_args(s)))
            self.launches += (hi > lo) + (s.n_items > 0) + (s.n_heavy > 0)
        if len(parts) > 1:
            s.relabel = None
            self.counts.copy_(self.slice_counts[:len(parts)].sum(0))
        flagged = None
        if flag_arcs and s.m >= FLAG_MIN_ARCS and DENSE_ARC_FRAC < 1.0:
            if self.flag_out is None:
                self.flag_out = torch.zeros(1, dtype=torch.int64, device=self.device)
            _lib.check(L.hb_sample_flagged_arcs(s.m, s.succ_buf.data_ptr(),
                                                self.chg_now.data_ptr(), FLAG_SAMPLES, t,
                                                self.flag_out.data_ptr(),
                                                self.stream.cuda_stream),
                       "hb_sample_flagged_arcs")
            self.launches += 1
            flagged = self.flag_out
        self.launches_at_last_step = self.launches
        nch, merged = (int(x) for x in self.counts.cpu())
        self.last_flagged = (int(flagged.item()) / FLAG_SAMPLES if flagged is not None
                             else None)
        self.last_nch = nch
        self.last_merged = merged
        self.merged_total += merged
        return nch

    def swap(self) -> None:
        self.cur, self.nxt = self.nxt, self.cur
        self.chg_prev, self.chg_now = self.chg_now, self.chg_prev
        self.prev_all = False
        self.full_pass = False

    def die_args(self) -> dict:
        """hb_step_args.die_head / die_rows / item_split (die-affine heavy items) when the
        schedule is eligible (schedule.die_eligible), every id is on the device and the
        device splits into two L2 dies.  First use per schedule: allocate the head buffer,
        map its chunks (hb_die_map) and reorder the ids inside the items
        (hb_die_partition); later runs on the same schedule reuse it."""
        s = self.sched
        if not (s.n_items > 0 and s.hot_rows > 0 and die_eligible(self.n, self.b, s.order)
                and s.partial.shape[0] >= 2 * s.n_items) or s.pending:
            return {}
        if _os.environ.get("HB_DIE", "0") != "1":     # opt-in
            return {}
        if s.die is None:
            L = _lib.hb()
            mb = int(_os.environ.get("HB_DIE_HEAD_MB", "112"))
            rows = min(s.hot_rows, (mb << 20) >> self.b)
            nbytes = rows << self.b
            s.die = False
            if nbytes >= 4096 and s.item_arcs <= 512:
                head = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
                bits = torch.zeros(int(L.hb_die_map_words(head.data_ptr(), nbytes)),
                                   dtype=torch.int32, device=self.device)
                stats = (ctypes.c_int64 * 4)()
                st = self.stream.cuda_stream
                _lib.check(L.hb_die_map(head.data_ptr(), nbytes, bits.data_ptr(), stats, st),
                           "hb_die_map")
                if stats[0] > 0:
                    split = torch.empty(s.n_items, dtype=torch.int32, device=self.device)
                    _lib.check(L.hb_die_partition(
                        s.n_items, s.item_node.data_ptr(), s.item_beg.data_ptr(),
                        s.offsets_ptr(), s.succ_buf.data_ptr(), s.item_arcs, self.b,
                        head.data_ptr(), rows, bits.data_ptr(), split.data_ptr(), st),
                        "hb_die_partition")
                    s.die = (head, rows, split, tuple(stats))
        if not s.die:
            return {}
        return dict(die_head=s.die[0].data_ptr(), die_rows=s.die[1],
                    item_split=s.die[2].data_ptr())


class _IdentityOrder:
    """Node order of the exact backend: original ids, the CSR uploaded as is."""

    perm = None
    rank = None

    def __init__(self, g, device: torch.device):
        off, suc = _graph_arrays(g)
        if not isinstance(off, torch.Tensor):
            off, suc = torch.from_numpy(np.array(off)), torch.from_numpy(np.array(suc))
        self.offsets = off.to(device=device, dtype=torch.int64).contiguous()
        self.succ = suc.to(device=device, dtype=torch.int32).contiguous()
        self.n = int(self.offsets.numel()) - 1

    @staticmethod
    def to_internal(x):
        return x

    @staticmethod
    def to_original(x):
        return x


class _ExactDevice(_Device):
    """Device state of the exact backend (engine.py:178-213): one bitset row of n bits per
    node (the reference's MSB-first bytes, padded to a 16-byte stride), OR-union and
    weighted popcount in hb_exact_union_step.  Identity node order; no frontier mode."""

    def __init__(self, g, config: HyperBallConfig):
        self.params = config.params
        self.b = config.params.b
        self.device = _resolve_device(config.device)
        self.stream = torch.cuda.current_stream(self.device)
        self.order = "identity"
        self.world, self.rank_id = 1, 0
        self._build_graph(g)
        n = self.n
        self.row_bytes = (n + 7) // 8
        self.row_stride = max(16, (self.row_bytes + 15) // 16 * 16)
        self.p = self.row_stride                    # row length of cur / nxt in bytes
        words = max((n + 31) // 32, 1)
        dv = self.device
        self.cur = torch.zeros((n, self.row_stride), dtype=torch.uint8, device=dv)
        self.nxt = torch.zeros((n, self.row_stride), dtype=torch.uint8, device=dv)
        self.chg_prev = torch.full((words,), -1, dtype=torch.int32, device=dv)
        self.chg_now = torch.zeros((words,), dtype=torch.int32, device=dv)
        self.est = torch.zeros(n, dtype=torch.float64, device=dv)
        self.counts = torch.zeros(2, dtype=torch.int64, device=dv)
        self.weights = np.ones(n, dtype=np.int64)
        self._w_dev = None
        self.merged_total = 0
        self.prev_all = True
        self.full_pass = True
        self.launches = 0
        self.launches_at_last_step = 0
        self.frontier = False
        self.fwd = None
        self.active = None
        self.last_nch = None

    def fresh(self, config: HyperBallConfig) -> "_ExactDevice":
        other = super().fresh(config)
        other.cur = torch.zeros_like(self.cur)
        other.nxt = torch.zeros_like(self.nxt)
        return other

    def _build_graph(self, g) -> None:
        self.sched = _IdentityOrder(g, self.device)
        self.n = self.sched.n
        self.graph_key = _graph_key(g)

    def seed(self, weights: np.ndarray | None) -> None:
        if weights is not None:
            self.weights = np.ascontiguousarray(weights, dtype=np.int64)
            self._w_dev = torch.from_numpy(self.weights).to(self.device)
        else:
            self.weights, self._w_dev = np.ones(self.n, dtype=np.int64), None
        _lib.check(_lib.hb().hb_exact_seed(
            self.n, self.row_stride, self.cur.data_ptr(), self.est.data_ptr(),
            self._w_dev.data_ptr() if self._w_dev is not None else None,
            self.stream.cuda_stream), "hb_exact_seed")
        self.launches += 1 if self.n else 0

    def set_weights(self, weights: np.ndarray) -> None:
        """Weights of a loaded checkpoint (no re-seed)."""
        self.weights = np.ascontiguousarray(weights, dtype=np.int64)
        ones = self.n == 0 or bool((self.weights == 1).all())
        self._w_dev = None if ones else torch.from_numpy(self.weights).to(self.device)

    def _frontier_ptr(self, dense: bool):
        return None

    def union_step(self, t: int, dense: bool, sums: _DeviceSums | None, peers=None,
                   clear_chg_now: bool = True, flag_arcs: bool = False) -> int:
        if peers is not None:
            raise ValueError("the exact backend runs on one device")
        s = self.sched
        sd = sums.sum_dist.data_ptr() if sums is not None else None
        sr = sums.sum_recip.data_ptr() if sums is not None else None
        dargs = sums.disc_args(t) if hasattr(sums, "disc_args") else (None, 0, 0, None, 0)
        _lib.check(_lib.hb().hb_exact_union_step(
            self.n, s.offsets.data_ptr(), s.succ.data_ptr(), self.cur.data_ptr(),
            self.nxt.data_ptr(), self.row_stride, self.chg_prev.data_ptr(),
            self.chg_now.data_ptr(), self.est.data_ptr(), sd, sr, t, int(dense),
            self._w_dev.data_ptr() if self._w_dev is not None else None, *dargs,
            self.counts.data_ptr(), self.counts.data_ptr() + 8, self.stream.cuda_stream),
            "hb_exact_union_step")
        self.launches += 1
        self.launches_at_last_step = self.launches
        nch, merged = (int(x) for x in self.counts.cpu())
        self.last_nch = nch
        self.last_merged = merged
        self.merged_total += merged
        return nch


def _make_device(g, config: HyperBallConfig) -> _Device:
    if config.backend == BACKEND_EXACT:
        return _ExactDevice(g, config)
    return _Device(g, config)



class HyperBallState:
    """Engine state resident on the device; host views are copies in original node order.

    At the end of iteration t, counter v holds the radius-t ball around v, ``est[v]`` its
    size estimate and ``changed_prev[v]`` whether v's counter moved in iteration t.
    """

    def __init__(self, config: HyperBallConfig, n: int, dev: _Device | None):
        self.config = config
        self.n = n
        self.t = 0
        self.num_changed = n
        self._dev = dev
        self._sums: _DeviceSums | None = None

    # host views -------------------------------------------------------------
    @property
    def est(self) -> np.ndarray:
        if self._dev is None:
            return np.zeros(0, dtype=np.float64)
        return self._dev.to_host(self._dev.est)

    def estimates(self) -> np.ndarray:
        """Current per-node ball-size estimates (a copy)."""
        return self.est

    @property
    def changed_prev(self) -> np.ndarray:
        if self._dev is None:
            return np.zeros(0, dtype=np.bool_)
        d = self._dev
        return d.to_host(unpack_bits(d.chg_prev, d.n))

    @property
    def _exact(self) -> bool:
        return self.config.backend == BACKEND_EXACT

    def register_matrix(self) -> np.ndarray:
        """Host copy of the working counter rows, original order, read-only: uint8 [n, p]
        registers, or for the exact backend the [n, ceil(n/8)] bitset rows."""
        if self._dev is None:
            width = (self.n + 7) // 8 if self._exact else self.config.params.p
            m = np.zeros((0, width), dtype=np.uint8)
        elif self._exact:
            d = self._dev
            m = np.ascontiguousarray(d.to_host(d.cur)[:, :d.row_bytes])
        else:
            m = self._dev.to_host(self._dev.cur)
        m.setflags(write=False)
        return m

    def counters(self) -> CounterArray:
        """Bit-packed snapshot of the current counters (probabilistic only), packed on the
        device (hb_pack_registers) in original node order."""
        if self._exact:
            raise ValueError("packed counters exist only for the probabilistic backend")
        pr = self.config.params
        if self._dev is None or self.n == 0:
            return CounterArray.from_dense(self.register_matrix(), pr)
        d = self._dev
        out = torch.empty((self.n, pr.row_bytes), dtype=torch.uint8, device=d.device)
        rank = d.sched.rank
        _lib.check(_lib.hb().hb_pack_registers(
            self.n, pr.b, pr.register_width, d.cur.data_ptr(),
            rank.data_ptr() if rank is not None else None, out.data_ptr(),
            d.stream.cuda_stream), "hb_pack_registers")
        return CounterArray(self.n, pr, d.to_host_raw(out).copy())

    def ball_members(self, v: int) -> np.ndarray:
        """Exact backend: the node ids in v's current ball (engine.py:209-211)."""
        if not self._exact:
            raise ValueError("ball members exist only for the exact backend")
        return np.flatnonzero(np.unpackbits(self.register_matrix()[v])[:self.n])

    def _exact_weights(self) -> np.ndarray:
        if self._dev is not None:
            return np.asarray(self._dev.weights, dtype=np.int64)
        return np.asarray(self._host[3], dtype=np.int64)

    @property
    def kernel_launches(self) -> int:
        return 0 if self._dev is None else self._dev.launches

    # checkpointing (engine.py:254-280, HBCK v1, both kinds) ---------------------
    def save(self, path) -> None:
        pr = self.config.params
        if self._exact:
            blob_cur, blob_nxt, kind = self.register_matrix().tobytes(), b"", 1
        else:
            blob_cur = self.counters().to_blob()
            blob_nxt, kind = CounterArray(self.n, pr).to_blob(), 0
        buf = io.BytesIO()
        buf.write(CHECKPOINT_MAGIC)
        buf.write(struct.pack("<HBQQQ", CHECKPOINT_VERSION, kind, self.n, self.t,
                              self.num_changed))
        buf.write(struct.pack("<BBQ", pr.b, pr.register_width, pr.seed & ((1 << 64) - 1)))
        for blob in (blob_cur, blob_nxt):
            buf.write(struct.pack("<Q", len(blob)))
            buf.write(blob)
        buf.write(self.changed_prev.astype(np.bool_).tobytes())
        buf.write(self.est.astype(np.float64).tobytes())
        if self._exact:
            buf.write(self._exact_weights().tobytes())
        with open(path, "wb") as fh:
            fh.write(buf.getvalue())


# ---------------------------------------------------------------------------- API

def initialize(g, config: HyperBallConfig) -> HyperBallState:
    """Seed one counter per node with item (v, 1) (or its weight replicas) on the device."""
    off = g.offsets
    n = (off.numel() if isinstance(off, torch.Tensor) else np.asarray(off).shape[0]) - 1
    w = _weights_array(config.weights, n)
    if w is not None:
        _check_weighted_width(config.params, w)
    if config.backend == BACKEND_EXACT:
        dev = _ExactDevice(g, config)
        dev.seed(w)
    else:                        # seeded while the successor ids are still uploading
        dev = _Device(g, config, seed_weights=w)
    return HyperBallState(config, n, dev)


def _split_observers(state: HyperBallState, observers):
    fused, generic = None, []
    for obs in observers:
        if fused is None and fusable(obs, state.n):
            fused = obs
        else:
            generic.append(obs)
    return fused, generic


def _bind_sums(state: HyperBallState, acc) -> _DeviceSums | None:
    dev = state._dev
    if acc is None:
        return None
    cur = state._sums
    if cur is not None and cur.acc is acc and cur.dev is dev and cur.still_valid():
        return cur
    if cur is not None and cur.dirty and cur.acc is not acc and cur.acc is not None:
        cur.pull_into(cur.acc)
    if isinstance(acc, CentralityAccumulator) and acc._binding is not None:
        if acc._binding.dirty and not acc._binding.stale:
            acc._binding.pull_into(acc)
        acc._binding = None
    sums = _DeviceSums(dev, acc)
    if isinstance(acc, CentralityAccumulator):
        acc._binding = sums
    state._sums = sums
    return sums


def iterate(g, state: HyperBallState, observers: Iterable = ()) -> int:
    """One synchronous ball-growth step on the device; returns how many counters changed."""
    if isinstance(state, _PendingState):
        state._attach(g)
    dev = state._dev
    t_next = state.t + 1
    observers = list(observers)
    if state.n == 0 or dev is None:
        for obs in observers:
            obs.on_step(t_next, np.zeros(0), np.zeros(0))
        state.t = t_next
        state.num_changed = 0
        return 0
    old_sched = dev.bind_graph(g)
    if old_sched is not None and state._sums is not None:
        state._sums.reorder(old_sched, dev.sched)
    fused, generic = _split_observers(state, observers)
    sums = _bind_sums(state, fused)
    old = dev.est.clone() if generic else None
    # Merging an unchanged source is a no-op, so when nearly every counter
    # changed last iteration the step skips the per-source bitmap tests (dense mode):
    # identical bits, less work per arc.
    skip = state.config.skip_stable_nodes
    dense = (dev.prev_all or not skip
             or (dev.last_nch is not None and dev.last_nch >= DENSE_FRAC * dev.n))
    # (wide rows make a redundant merge dearer than the per-source test it saves: the
    # measured 0.7 is for p = 16; from p = 128 up the rule waits for 0.9)
    arc_frac = DENSE_ARC_FRAC if state.config.params.p <= 64 else max(DENSE_ARC_FRAC, 0.9)
    arc_dense = (not dense and getattr(dev, "last_flagged", None) is not None
                 and dev.last_flagged >= arc_frac)
    nch = dev.union_step(t_next, dense or arc_dense, sums, flag_arcs=skip)
    if generic:
        old_h, new_h = dev.to_host(old), dev.to_host(dev.est)
        old_h.setflags(write=False)
        new_h.setflags(write=False)
        for obs in generic:
            obs.on_step(t_next, old_h, new_h)
    dev.swap()
    if sums is not None:
        sums.dirty = True
        if sums.foreign:
            sums.pull_into(sums.acc)
    state.t = t_next
    state.num_changed = nch
    return nch


def run(g, config: HyperBallConfig, observers: Iterable = ()) -> HyperBallState:
    """Initialize and iterate until no counter changes (engine.py:402-410)."""
    state = initialize(g, config)
    return resume(g, state, observers)


def resume(g, state: HyperBallState, observers: Iterable = ()) -> HyperBallState:
    """Continue a (possibly checkpointed) run to convergence (engine.py:413-435)."""
    cfg = state.config
    observers = list(observers)
    if state.n > 0:
        while True:
            started = time.perf_counter()
            nch = iterate(g, state, observers)
            if cfg.progress is not None:
                elapsed_ms = (time.perf_counter() - started) * 1000.0
                cfg.progress.write(f"t={state.t} changed={nch} elapsed_ms={elapsed_ms:.0f}\n")
            if nch == 0:
                break
            if cfg.max_iterations is not None and state.t >= cfg.max_iterations:
                raise ConvergenceError(state.t, nch)
    else:
        state.num_changed = 0
    # The fused accumulator keeps the final estimates on the device (its coreach is
    # downloaded on first read); any other observer gets the host copy as in the reference.
    sums = state._sums
    fused = (sums.acc if sums is not None and not sums.stale and not sums.foreign
             and sums.dev is state._dev else None)
    if fused is not None and any(o is fused for o in observers) and all(
            o is fused for o in observers):
        fused._converged_on_device(sums.fetch_coreach)
        return state
    final = state.est
    final.setflags(write=False)
    for obs in observers:
        obs.on_converged(final)
    return state


def load_state(path, config: HyperBallConfig | None = None, graph=None) -> HyperBallState:
    """Rebuild a saved HBCK v1 state (engine.py:283-327).  The device half is attached on
    the first ``iterate``/``resume`` with the graph (or immediately when `graph` is given)."""
    with open(path, "rb") as fh:
        data = fh.read()
    if data[:4] != CHECKPOINT_MAGIC:
        raise ValueError("bad checkpoint magic")
    version, kind, n, t, num_changed = struct.unpack("<HBQQQ", data[4:31])
    if version != CHECKPOINT_VERSION:
        raise ValueError(f"unsupported checkpoint version {version}")
    if kind not in (0, 1):
        raise ValueError(f"unknown checkpoint kind {kind}")
    b, width, seed = struct.unpack("<BBQ", data[31:41])
    params = CounterParams(b=b, register_width=width, seed=seed)
    pos = 41
    blobs = []
    for _ in range(2):
        (length,) = struct.unpack("<Q", data[pos:pos + 8])
        pos += 8
        blobs.append(data[pos:pos + length])
        pos += length
    changed_prev = np.frombuffer(data, dtype=np.bool_, count=n, offset=pos).copy()
    pos += n
    est = np.frombuffer(data, dtype=np.float64, count=n, offset=pos).copy()
    pos += 8 * n
    weights = None
    if kind == 0:
        dense = CounterArray.from_blob(blobs[0])     # unpacked on the device in _attach
    else:
        weights = np.frombuffer(data, dtype=np.int64, count=n, offset=pos).copy()
        dense = np.frombuffer(blobs[0], dtype=np.uint8).reshape(n, (n + 7) // 8).copy()
    if config is None:
        config = HyperBallConfig(params=params, weights=weights,
                                 backend=BACKEND_PROBABILISTIC if kind == 0 else BACKEND_EXACT)
    elif (config.backend == BACKEND_EXACT) != (kind == 1):
        raise ValueError(f"checkpoint kind {kind} does not match backend {config.backend!r}")
    state = _PendingState(config, n, (dense, changed_prev, est, weights))
    state.t = t
    state.num_changed = num_changed
    if graph is not None:
        state._attach(graph)
    return state


class _PendingState(HyperBallState):
    """A loaded state whose device half is created once the graph is known."""

    def __init__(self, config, n, host):
        super().__init__(config, n, None)
        self._host = host

    def _attach(self, g) -> None:
        if self._dev is not None:
            return
        dense, changed_prev, est, weights = self._host
        dev = _make_device(g, self.config)
        if dev.n != self.n:
            raise ValueError(f"graph has {dev.n} nodes, checkpoint has {self.n}")
        if isinstance(dense, CounterArray):           # packed registers: unpack on device
            pr = dense.params
            packed = torch.from_numpy(np.ascontiguousarray(dense.registers)).to(dev.device)
            cur = torch.empty((self.n, pr.p), dtype=torch.uint8, device=dev.device)
            perm = dev.sched.perm
            if self.n:
                _lib.check(_lib.hb().hb_unpack_registers(
                    self.n, pr.b, pr.register_width, packed.data_ptr(),
                    perm.data_ptr() if perm is not None else None, cur.data_ptr(),
                    dev.stream.cuda_stream), "hb_unpack_registers")
            del packed
            dev.cur = cur
            dev.nxt = cur.clone()
            dev.est = dev.to_internal(torch.from_numpy(est))
            dev.chg_prev = pack_bits(dev.to_internal(torch.from_numpy(changed_prev)))
        else:
            if weights is not None:
                dev.set_weights(weights)
                padded = np.zeros((self.n, dev.row_stride), dtype=np.uint8)
                padded[:, :dense.shape[1]] = dense
                dense = padded
            cur = torch.from_numpy(dense).to(dev.device)
            dev.restore_original(cur, cur.clone(), torch.from_numpy(est).to(dev.device),
                                 torch.from_numpy(changed_prev).to(dev.device))
        # the recycled buffer must hold the current rows (lazy double-buffer invariant)
        dev.nxt.copy_(dev.cur)
        dev.prev_all = bool(changed_prev.all()) if self.n else False
        dev.full_pass = True
        self._dev = dev
        self._host = None

    @property
    def est(self):
        if self._dev is None:
            return self._host[2].copy()
        return super().est

    @property
    def changed_prev(self):
        if self._dev is None:
            return self._host[1].copy()
        return super().changed_prev

    def register_matrix(self):
        if self._dev is None:
            h = self._host[0]
            m = h.to_dense() if isinstance(h, CounterArray) else h.copy()
            m.setflags(write=False)
            return m
        return super().register_matrix()

    def counters(self) -> CounterArray:
        if self._dev is None and isinstance(self._host[0], CounterArray):
            return self._host[0].copy()
        return super().counters()



def run_multi(g, config: HyperBallConfig, runs: int, discounts=(), observers_factory=None,
              batch: int | None = None):
    """The reference CLI's repeated runs (cli.py:222-254): run r uses seed config.seed + r
    and its own CentralityAccumulator.  Returns [(state, accumulator)]; feed finalize_* of
    each accumulator to multi_run_aggregate.

    batch: runs sharing one union pass (multirun.py; a power of two, batch * p <= 256).
    None picks multirun.batch_size (p = 16: 4, p = 32: 2, else 1).  Batching needs the
    probabilistic backend and at most 8 device-fusable discounts; otherwise, and for
    batch = 1, the runs go one after the other, the graph uploaded and scheduled once and
    only the counters re-seeded.  Either way every run's bits equal an independent run."""
    from dataclasses import replace
    from . import multirun
    if runs < 1:
        raise ValueError("runs must be >= 1")
    n = (g.offsets.numel() if isinstance(g.offsets, torch.Tensor)
         else np.asarray(g.offsets).shape[0]) - 1
    if batch is None:
        batch = multirun.batch_size(config.params.p, runs)
    if batch < 1:
        raise ValueError("batch must be >= 1")
    accs = [CentralityAccumulator(n, discounts) for _ in range(runs)]
    obs = [[accs[r]] + (list(observers_factory(r)) if observers_factory else [])
           for r in range(runs)]
    seeds = [config.params.seed + r for r in range(runs)]
    out = []
    dev = None
    r = 0
    while r < runs:
        k = min(batch, runs - r)
        k = 1 << (k.bit_length() - 1)                  # largest power of two <= k
        if k >= 2 and multirun.supported(config, k, discounts):
            states = multirun.run_batched(g, config, seeds[r:r + k], obs[r:r + k], discounts)
            out.extend(zip(states, accs[r:r + k]))
            r += k
            continue
        cfg = replace(config, params=replace(config.params, seed=seeds[r]))
        w = _weights_array(cfg.weights, n)
        if w is not None:
            _check_weighted_width(cfg.params, w)
        if dev is None:
            dev = _make_device(g, cfg)
        else:                               # same graph and schedule, fresh counters
            dev = dev.fresh(cfg)
        state = HyperBallState(cfg, n, dev)
        dev.seed(w)
        out.append((resume(g, state, obs[r]), accs[r]))
        r += 1
    return out
