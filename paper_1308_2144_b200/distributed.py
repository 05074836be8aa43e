"""Multi-GPU HyperBall: node-range partition + changed-row exchange.

Within an iteration every counter row depends only on the previous iteration's rows
(Jacobi double buffer, engine.py:393), so the node set is partitioned into contiguous
internal-id ranges, one per rank (schedule.partition_bounds; in degree order a
round-robin deal of the degree ranking).  Every rank keeps a full replica of the
register rows.  One iteration on rank r:

1. ``hb_union_step`` over its own range: owned rows of ``nxt``, owned change bits,
   estimates and fused accumulator sums.
2. ``hb_refresh_rows``: rows owned elsewhere that changed in the previous iteration are
   copied ``cur -> nxt`` (keeps the lazy double buffer valid for remote rows).
3. ``hb_gather_changed``: pack (id, row) of the owned rows that changed.
4. exchange: all-gather of the per-rank changed counts -- whose sum is the global
   termination count, i.e. the reference's ``nch = sum(f.result() ...)`` barrier
   (engine.py:390) as one collective -- then all-gather of the packed rows (padded to the
   largest count).
5. ``hb_scatter_rows``: write every other rank's rows into ``nxt`` and set their change
   bits, so the next iteration's source-skip bitmap is global.

The protocol is written once (``iterate_rank``) over a small rank-state interface, so the
same driver runs with NCCL on GPUs (``CudaRankState``), in one process over several
simulated ranks on one GPU (``run_simulated``, which exercises every exchange kernel),
and -- in the CPU test suite -- with gloo over an oracle-backed rank state.
"""

from __future__ import annotations

import time
from typing import Iterable

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .centrality import CentralityAccumulator, fusable
from .engine import (DENSE_FRAC, ConvergenceError, HyperBallConfig, _Device, _weights_array,
                     _check_weighted_width)


class TorchComm:
    """Collectives of one rank over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def exchange(self, ids: torch.Tensor, rows: torch.Tensor, k: int):
        """All-gather the packed changed rows.  Returns (total changed, [(ids_q, rows_q)]
        for every other rank q)."""
        dev = ids.device
        cnt = torch.tensor([k], dtype=torch.int64, device=dev)
        counts = [torch.zeros_like(cnt) for _ in range(self.world)]
        dist.all_gather(counts, cnt, group=self.group)
        counts = [int(c.item()) for c in counts]
        total = sum(counts)
        kmax = max(counts)
        if kmax == 0:
            return total, []
        p = rows.shape[1]
        send_ids = ids[:kmax] if ids.shape[0] >= kmax else torch.cat(
            [ids, ids.new_zeros(kmax - ids.shape[0])])
        send_rows = rows[:kmax] if rows.shape[0] >= kmax else torch.cat(
            [rows, rows.new_zeros((kmax - rows.shape[0], p))])
        all_ids = [torch.empty_like(send_ids) for _ in range(self.world)]
        all_rows = [torch.empty_like(send_rows) for _ in range(self.world)]
        dist.all_gather(all_ids, send_ids.contiguous(), group=self.group)
        dist.all_gather(all_rows, send_rows.contiguous(), group=self.group)
        parts = []
        for q in range(self.world):
            if q == self.rank or counts[q] == 0:
                continue
            parts.append((all_ids[q][:counts[q]], all_rows[q][:counts[q]]))
        return total, parts

    def all_gather_slices(self, x: torch.Tensor, lo: int, hi: int, n: int) -> torch.Tensor:
        """Every rank's [lo, hi) slice of a per-node array, assembled (internal order)."""
        dev = x.device
        bounds = torch.tensor([lo, hi], dtype=torch.int64, device=dev)
        allb = [torch.zeros_like(bounds) for _ in range(self.world)]
        dist.all_gather(allb, bounds, group=self.group)
        allb = [tuple(int(v) for v in b.tolist()) for b in allb]
        width = max(h - l for l, h in allb)
        send = torch.zeros((width,) + tuple(x.shape[1:]), dtype=x.dtype, device=dev)
        send[:hi - lo] = x[lo:hi]
        out = [torch.empty_like(send) for _ in range(self.world)]
        dist.all_gather(out, send, group=self.group)
        full = torch.empty((n,) + tuple(x.shape[1:]), dtype=x.dtype, device=dev)
        for (l, h), part in zip(allb, out):
            full[l:h] = part[:h - l]
        return full


class _RankSums:
    """A rank's fused accumulator sums (full-length arrays, the owned slice is live)."""

    def __init__(self, n: int, device, specs=()):
        self.specs = list(specs)
        self.sum_dist = torch.zeros(n, dtype=torch.float64, device=device)
        self.sum_recip = torch.zeros(n, dtype=torch.float64, device=device)
        self.disc = torch.zeros((len(self.specs), n), dtype=torch.float64, device=device)
        self.n = n

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
        return self.disc.data_ptr(), self.n, k, ctypes.cast(scale, ctypes.c_void_p), div


def _fill_accumulators(accs, host) -> None:
    """Hand the gathered sums (original order) to the fused accumulators."""
    for acc in accs:
        if isinstance(acc, CentralityAccumulator):
            acc._sum_dist, acc._sum_recip = host["sum_dist"].copy(), host["sum_recip"].copy()
            acc._discounted = {spec.name: host["disc:" + spec.name].copy()
                               for spec in acc.discounts}
            acc._fresh = False
        else:
            acc.sum_dist, acc.sum_recip = host["sum_dist"].copy(), host["sum_recip"].copy()


def _specs_of(accs):
    """Discount specs of the (single) fused accumulator; several fused accumulators must
    agree (they all receive the same sums)."""
    specs = None
    for acc in accs:
        mine = [d.name for d in getattr(acc, "discounts", [])]
        if specs is None:
            specs = list(getattr(acc, "discounts", []))
        elif [d.name for d in specs] != mine:
            raise ValueError("fused accumulators of one distributed run must carry the same "
                             "discounts")
    return specs or []


class CudaRankState:
    """One rank's device state: full register replica, owned range [lo, hi)."""

    def __init__(self, g, config: HyperBallConfig, world: int, rank: int, packed: bool = True):
        if config.backend != "probabilistic":
            raise ValueError("multi-GPU runs use the probabilistic backend; the exact bitset "
                             "backend is a single-device validation tool")
        n = (g.offsets.numel() if isinstance(g.offsets, torch.Tensor)
             else np.asarray(g.offsets).shape[0]) - 1
        w = _weights_array(config.weights, n)
        if w is not None:
            _check_weighted_width(config.params, w)
        self.dev = _Device(g, config, world=world, rank_id=rank)
        self.dev.seed(w)
        self.n, self.b, self.p = self.dev.n, self.dev.b, self.dev.p
        self.lo, self.hi = self.dev.sched.lo, self.dev.sched.hi
        cap = max(self.hi - self.lo, 1)
        dv = self.dev.device
        # rows travel 5-bit packed when every register fits (register_width <= 5)
        self.packed = int(config.params.register_width <= 5 and packed)
        self.row_bytes = (_lib.hb().hb_packed_row_bytes(self.b) if self.packed else self.p)
        self.ids_buf = torch.empty(cap, dtype=torch.int32, device=dv)
        self.rows_buf = torch.empty((cap, self.row_bytes), dtype=torch.uint8, device=dv)
        self.count = torch.zeros(1, dtype=torch.int64, device=dv)
        self.sums = None

    def bind_sums(self, specs=()):
        """Device sums of the fused accumulator, including its discounted gains
        (centrality.py:26-101,149-150; up to MAX_FUSED_DISCOUNTS, folded in the union
        epilogue like on one GPU)."""
        self.sums = _RankSums(self.n, self.dev.device, specs)
        return self.sums

    def local_step(self, t: int, dense: bool) -> int:
        return self.dev.union_step(t, dense, self.sums)

    def refresh_unowned(self) -> None:
        d = self.dev
        _lib.check(_lib.hb().hb_refresh_rows(self.n, self.lo, self.hi, d.chg_prev.data_ptr(),
                                             d.cur.data_ptr(), d.nxt.data_ptr(), self.b,
                                             d.stream.cuda_stream), "hb_refresh_rows")
        d.launches += 1

    def gather_changed(self):
        d = self.dev
        _lib.check(_lib.hb().hb_gather_changed(self.lo, self.hi, d.chg_now.data_ptr(),
                                               d.nxt.data_ptr(), self.b, self.packed,
                                               self.ids_buf.data_ptr(),
                                               self.rows_buf.data_ptr(),
                                               self.count.data_ptr(), d.stream.cuda_stream),
                   "hb_gather_changed")
        d.launches += 1
        k = int(self.count.item())
        return self.ids_buf[:k], self.rows_buf[:k], k

    def apply_remote(self, ids: torch.Tensor, rows: torch.Tensor) -> None:
        d = self.dev
        k = ids.shape[0]
        if k == 0:
            return
        _lib.check(_lib.hb().hb_scatter_rows(k, ids.data_ptr(), rows.contiguous().data_ptr(),
                                             self.b, self.packed, d.nxt.data_ptr(),
                                             d.chg_now.data_ptr(),
                                             d.stream.cuda_stream), "hb_scatter_rows")
        d.launches += 1

    def swap(self) -> None:
        self.dev.swap()

    # per-node arrays in internal order for the final gather
    def per_node(self):
        out = {"est": self.dev.est}
        if self.sums is not None:
            out["sum_dist"] = self.sums.sum_dist
            out["sum_recip"] = self.sums.sum_recip
            for i, spec in enumerate(self.sums.specs):
                out["disc:" + spec.name] = self.sums.disc[i]
        return out

    def to_original(self, x: torch.Tensor) -> np.ndarray:
        return self.dev.to_host(x)


def iterate_rank(state, comm, t: int, dense: bool) -> int:
    """One distributed iteration on one rank; returns the GLOBAL changed count."""
    state.local_step(t, dense)
    state.refresh_unowned()
    ids, rows, k = state.gather_changed()
    total, parts = comm.exchange(ids, rows, k)
    for ids_q, rows_q in parts:
        state.apply_remote(ids_q, rows_q)
    state.swap()
    return total


class DistributedResult:
    """What ``run_distributed`` returns on every rank (host arrays, original order)."""

    def __init__(self, t, num_changed, est, sum_dist=None, sum_recip=None, launches=0):
        self.t, self.num_changed, self.est = t, num_changed, est
        self.sum_dist, self.sum_recip = sum_dist, sum_recip
        self.kernel_launches = launches

    def estimates(self):
        return self.est.copy()


def setup_push(state: "CudaRankState", group=None):
    """Move the rank's buffers into symmetric memory for the fused push; None if the
    platform has no symmetric memory (the all-gather exchange is used instead)."""
    try:
        return SymmetricBuffers(state, group)
    except Exception as exc:   # no NVLink / symmetric memory: fall back, loudly
        import warnings
        warnings.warn(f"fused push unavailable ({exc!r}); using the all-gather exchange")
        return None


def iterate_push(state: "CudaRankState", symm: SymmetricBuffers, t: int, dense: bool,
                 group=None) -> int:
    """One fused-push iteration: union epilogue stores into the peers, then one NCCL
    all-reduce of the changed count -- the termination test (engine.py:390) and the
    barrier after which every rank's pushed rows are visible -- then (packed push) the
    rows the peers wrote are unpacked from this step's inbox, then swap."""
    peer_nxt, peer_chg = symm.peer_pointers(state.dev, t)
    nch = push_step(state, t, dense, peer_nxt, peer_chg, symm.pstride, symm.prev_copy)
    tot = torch.tensor([nch], dtype=torch.int64, device=state.dev.device)
    dist.all_reduce(tot, group=group)
    if symm.pstride:
        unpack_inbox(state, symm.inbox_of(t), symm.prev_copy)
    state.swap()
    return int(tot.item())


def unpack_inbox(state: "CudaRankState", inbox: torch.Tensor, prev_copy: torch.Tensor) -> None:
    """Packed push, receiver side (after the step's barrier), rows of the other ranks:
    changed this step -> unpacked from `inbox`; changed in the previous step only -> nxt =
    cur (the lazy double buffer, refreshed locally)."""
    d = state.dev
    _lib.check(_lib.hb().hb_unpack_inbox(d.n, state.lo, state.hi, d.b, d.chg_now.data_ptr(),
                                         prev_copy.data_ptr(), inbox.data_ptr(),
                                         d.cur.data_ptr(), d.nxt.data_ptr(),
                                         d.stream.cuda_stream),
               "hb_unpack_inbox")
    d.launches += 1


def run_distributed(g, config: HyperBallConfig, observers: Iterable = (), group=None,
                    state_factory=None, exchange: str = "push") -> DistributedResult:
    """``run`` (engine.py:402-435) over every rank of `group`; call it on every rank with
    the same graph.  exchange="push" (default on NCCL) fuses the row exchange into the
    union epilogue over symmetric memory; "allgather" packs, all-gathers and scatters the
    changed rows.  Fused ``CentralityAccumulator`` observers are supported (filled on every
    rank after convergence); other observers get ``on_converged`` only."""
    comm = TorchComm(group)
    factory = state_factory or (lambda: CudaRankState(g, config, comm.world, comm.rank))
    st = factory()
    observers = list(observers)
    accs = [o for o in observers if fusable(o, st.n)]
    if accs:
        st.bind_sums(_specs_of(accs))
    symm = None
    if (exchange == "push" and comm.world > 1 and isinstance(st, CudaRankState)
            and dist.get_backend(group) == "nccl" and st.n > 0):
        symm = setup_push(st, group)
    t = 0
    nch = st.n
    if st.n > 0:
        while True:
            started = time.perf_counter()
            dense = (t == 0 or not config.skip_stable_nodes
                     or nch >= DENSE_FRAC * st.n)   # every rank sees the same global nch
            if symm is not None:
                nch = iterate_push(st, symm, t + 1, dense, group)
            else:
                nch = iterate_rank(st, comm, t + 1, dense)
            t += 1
            if config.progress is not None and comm.rank == 0:
                config.progress.write(f"t={t} changed={nch} elapsed_ms="
                                      f"{(time.perf_counter() - started) * 1000.0:.0f}\n")
            if nch == 0:
                break
            if config.max_iterations is not None and t >= config.max_iterations:
                raise ConvergenceError(t, nch)
    else:
        nch = 0
    arrays = {k: comm.all_gather_slices(v, st.lo, st.hi, st.n) for k, v in st.per_node().items()}
    dev_ = getattr(st, "dev", None)
    mt = torch.tensor([getattr(dev_, "merged_total", 0)], dtype=torch.int64,
                      device=arrays["est"].device)
    dist.all_reduce(mt, group=group)
    host = {k: st.to_original(v) for k, v in arrays.items()}
    res = DistributedResult(t, nch, host["est"], host.get("sum_dist"), host.get("sum_recip"),
                            getattr(dev_, "launches", 0))
    res.merged_total = int(mt.item())
    final = host["est"]
    final.setflags(write=False)
    _fill_accumulators(accs, host)
    for obs in observers:
        obs.on_converged(final)
    return res


# ---------------------------------------------------------------- fused push exchange

def _ptr_array(ptrs):
    import ctypes
    arr = (ctypes.c_void_p * max(len(ptrs), 1))(*ptrs)
    return arr


def push_step(state: "CudaRankState", t: int, dense: bool, peer_nxt, peer_chg,
              pstride: int = 0, prev_copy: torch.Tensor | None = None) -> int:
    """Union step whose epilogue stores this rank's written rows and change bits straight
    into every peer's replica (hb_union_step with peers) -- or, with pstride > 0, into
    the peers' inboxes 5-bit packed (peer_nxt are then inbox addresses).  Afterwards this
    rank's chg_prev is cleared: it becomes chg_now of the next step, into which peers may
    push only after the barrier that follows; a packed push first keeps a copy of it
    (prev_copy) for the unpack after the barrier.  Returns the LOCAL changed count."""
    d = state.dev
    n_peers = len(peer_nxt)
    nch = d.union_step(t, dense, state.sums,
                       peers=(n_peers, _ptr_array(peer_nxt), _ptr_array(peer_chg), pstride),
                       clear_chg_now=False)
    if pstride:
        prev_copy.copy_(d.chg_prev)
    d.chg_prev.zero_()
    return nch


def packed_push_stride(state: "CudaRankState", packed: bool = True) -> int:
    """Bytes per inbox row of the packed push (0 = rows travel unpacked): 5-bit fields need
    every register < 32, i.e. register_width <= 5."""
    if not packed or state.dev.params.register_width > 5:
        return 0
    return int(_lib.hb().hb_push_row_stride(state.dev.b))


class SymmetricBuffers:
    """The register double buffer and the two change bitmaps of one rank in symmetric
    memory (torch.distributed._symmetric_memory): every peer maps them, so the union
    epilogue can store into them over NVLink.  With the packed push (register_width <=
    5) the peers store 5-bit packed rows into a double-buffered inbox instead (step t
    uses inbox t % 2: a peer one step ahead writes the other one), and this rank unpacks
    them after the step's barrier -- 37.5% fewer NVLink bytes per row (25% at p = 16)."""

    def __init__(self, state: "CudaRankState", group=None, packed: bool = True):
        import torch.distributed._symmetric_memory as symm
        d = state.dev
        n, p = d.n, d.p
        words = d.chg_prev.numel()
        self.pstride = packed_push_stride(state, packed)
        gname = group.group_name if group is not None else dist.group.WORLD.group_name
        if self.pstride:
            self.inbox = symm.empty((2, n, self.pstride), dtype=torch.uint8, device=d.device)
            self.h_inbox = symm.rendezvous(self.inbox, gname)
            self.prev_copy = torch.zeros_like(d.chg_prev)
        else:
            self.inbox = self.h_inbox = self.prev_copy = None
        self.regs = symm.empty((2, n, p), dtype=torch.uint8, device=d.device)
        self.bits = symm.empty((2, words), dtype=torch.int32, device=d.device)
        self.regs[0].copy_(d.cur)
        self.regs[1].copy_(d.nxt)      # seeded rows the first iteration may skip (_Device.seed)
        self.bits[0].copy_(d.chg_prev)
        self.bits[1].zero_()
        d.cur, d.nxt = self.regs[0], self.regs[1]
        d.chg_prev, d.chg_now = self.bits[0], self.bits[1]
        self.h_regs = symm.rendezvous(self.regs, gname)
        self.h_bits = symm.rendezvous(self.bits, gname)
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def inbox_of(self, t: int) -> torch.Tensor:
        return self.inbox[t & 1]

    def peer_pointers(self, d, t: int = 0):
        """Peer addresses the union epilogue of step t stores into: their nxt buffers (or
        their step-t inboxes, packed) and their chg_now bitmaps."""
        oc = d.chg_now.data_ptr() - self.bits.data_ptr()
        qs = [q for q in range(self.world) if q != self.rank]
        if self.pstride:
            oi = self.inbox_of(t).data_ptr() - self.inbox.data_ptr()
            rows = [int(self.h_inbox.buffer_ptrs[q]) + oi for q in qs]
        else:
            on = d.nxt.data_ptr() - self.regs.data_ptr()
            rows = [int(self.h_regs.buffer_ptrs[q]) + on for q in qs]
        return rows, [int(self.h_bits.buffer_ptrs[q]) + oc for q in qs]


def run_simulated(g, config: HyperBallConfig, world: int, observers: Iterable = (),
                  packed: bool = True, exchange: str = "allgather"):
    """All `world` ranks in one process on one GPU, phase by phase (no kernel waits on
    another rank).  Exercises the partition and every exchange kernel; results must be
    bit-identical to the single-GPU run."""
    states = [CudaRankState(g, config, world, r, packed) for r in range(world)]
    pstride = packed_push_stride(states[0], packed) if exchange == "push" else 0
    inboxes, prev_copies = {}, {}
    if pstride:
        for s in states:
            inboxes[id(s)] = torch.empty((2, s.n, pstride), dtype=torch.uint8,
                                         device=s.dev.device)
            prev_copies[id(s)] = torch.zeros_like(s.dev.chg_prev)
    observers = list(observers)
    accs = [o for o in observers if fusable(o, states[0].n)]
    if accs:
        specs = _specs_of(accs)
        for s in states:
            s.bind_sums(specs)
    t = 0
    nch = states[0].n
    if nch > 0:
        while True:
            dense = (t == 0 or not config.skip_stable_nodes
                     or nch >= DENSE_FRAC * states[0].n)
            if exchange == "push":
                # every rank's epilogue writes into the other ranks' buffers (or packed
                # inboxes); the ranks run one after another, so no kernel ever waits on
                # another; the packed rows are unpacked once every rank has pushed
                nch = 0
                for s in states:
                    peers = [q for q in states if q is not s]
                    if pstride:
                        rows = [inboxes[id(q)][(t + 1) & 1].data_ptr() for q in peers]
                    else:
                        rows = [q.dev.nxt.data_ptr() for q in peers]
                    nch += push_step(s, t + 1, dense, rows,
                                     [q.dev.chg_now.data_ptr() for q in peers], pstride,
                                     prev_copies.get(id(s)))
                if pstride:
                    for s in states:
                        unpack_inbox(s, inboxes[id(s)][(t + 1) & 1], prev_copies[id(s)])
            else:
                for s in states:
                    s.local_step(t + 1, dense)
                    s.refresh_unowned()
                packed_rows = [s.gather_changed() for s in states]
                nch = sum(k for _, _, k in packed_rows)
                for r, s in enumerate(states):
                    for q, (ids, rows, k) in enumerate(packed_rows):
                        if q != r and k:
                            s.apply_remote(ids, rows)
            for s in states:
                s.swap()
            t += 1
            if nch == 0:
                break
            if config.max_iterations is not None and t >= config.max_iterations:
                raise ConvergenceError(t, nch)
    n = states[0].n
    full = {}
    for key in states[0].per_node():
        x = torch.empty_like(states[0].per_node()[key])
        for s in states:
            x[s.lo:s.hi] = s.per_node()[key][s.lo:s.hi]
        full[key] = states[0].to_original(x)
    res = DistributedResult(t, nch, full["est"], full.get("sum_dist"), full.get("sum_recip"),
                            sum(s.dev.launches for s in states))
    res.registers = [s.to_original(s.dev.cur) for s in states]
    final = full["est"]
    _fill_accumulators(accs, full)
    for obs in observers:
        obs.on_converged(final)
    return res
