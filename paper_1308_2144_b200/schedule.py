"""Device-resident graph in schedule order, plus the heavy-node work split.

The reference walks nodes in id order with one CPU thread per arc-balanced range
(engine.py:351-390).  On the B200 the union kernel assigns lane groups to nodes, so the
schedule decides:

* ``order``: ``identity`` keeps node ids; ``window`` keeps them inside the light
  kernel's grid-stride chunks but sorts each chunk by in-degree (best when ids carry
  locality, e.g. config 4's +-1024 window, and in-degrees vary); ``degree`` relabels nodes by descending
  in-degree (stable), so every warp sees neighbours of equal degree, hubs sit first and
  their hot register rows share cache lines, and zero in-degree nodes trail.  The
  relabelling is internal: hashes use original ids and every host-visible array is
  returned in original order, so registers stay bit-identical.
* ``heavy`` nodes (in-degree above ``light_max_deg``) are cut into work items of
  ``item_arcs`` arcs; one warp merges an item into a partial row, a second pass merges
  the partial rows of a node and runs the epilogue.
"""

from __future__ import annotations

import os
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib


def hot_head_rows(n: int, order: str, world: int) -> int:
    """Rows of the L2-protected hot head (hb_step_args.hot_rows).  In degree order on one
    GPU the most-read rows are the first rows.  With world > 1 the degree deal gives every
    rank a contiguous range that starts with ITS share of them, so the hot set is W
    sub-heads and the single protected range [0, H) covers one rank's sub-head while every
    other rank's hot rows are marked evict-first: measured per rank on one GPU
    (tools/rank_step_bench.py, config 5 dense step, rank 0 of W = 2 / 4 / 8): 18.0 / 10.7 /
    6.1 ms with the range, 18.6 / 9.4 / 4.8 ms without any hint -- off from 3 ranks up."""
    return n if order == "degree" and world <= 2 else 0


def die_eligible(n: int, b: int, order: str) -> bool:
    """Can hb_union_step_v2 use die-affine heavy items on this schedule?  (16- / 32-register
    rows of a register array >= 1 GB in degree order: include/hyperball_b200.h, die_bits.)"""
    if os.environ.get("HB_DIE", "0") != "1":        # opt-in
        return False
    min_mb = int(os.environ.get("HB_DIE_MIN_MB", "1024"))
    return order == "degree" and b <= 5 and (n << b) >= (min_mb << 20)


@dataclass
class Schedule:
    n: int
    m: int
    b: int
    order: str
    perm: torch.Tensor | None      # int32 [n]: internal id -> original id
    rank: torch.Tensor | None      # int32 [n]: original id -> internal id
    offsets: torch.Tensor          # int64 [n+1], internal ids
    succ_buf: torch.Tensor         # int32 [m], internal ids (see `succ`)
    lo: int
    hi: int
    light_lo: int
    light_hi: int
    light_hi_steady: int           # light_hi once zero in-degree nodes can no longer change
    light_max_deg: int
    item_arcs: int
    heavy_nodes: torch.Tensor
    item_first: torch.Tensor
    finish_order: torch.Tensor     # int32 [n_heavy]: heavy indices, mega nodes first
    n_mega: int                    # heavy nodes merged one warp per node
    item_node: torch.Tensor
    item_beg: torch.Tensor
    partial: torch.Tensor
    max_deg: int
    hot_rows: int = 0              # degree order: head of the rows kept persisting in L2
    die: object = None             # die-affine items: None = not tried, False = off, else
                                   # (head buffer, rows, item_split, hb_die_map stats)
    # Streamed upload (window / identity order): row slices [r0, r1) whose successor ids
    # are still in flight on the side stream (event) and, for the window order, not yet
    # relabelled (relabel = (old offsets, old ids, perm, rank)).  Iteration 1 consumes them
    # slice by slice (engine._Device.union_step); any other reader of `succ` first
    # finishes them all on `stream`.
    pending: list = field(default_factory=list)
    relabel: tuple | None = None
    stream: object = None
    # Rank-local CSR (multi-GPU): `offsets` / `succ_buf` hold only the rows this rank owns
    # (offsets[i] is the local position of row row_base + i; rows row_base..lo-1 are
    # empty padding); kernels index offsets by global internal id through offsets_ptr()
    # (base shifted by row_base rows), valid for every id they touch.  Passes over every row (frontier marking,
    # forward graph) are not available on a local CSR.
    row_base: int = 0
    local: bool = False

    def offsets_ptr(self) -> int:
        return self.offsets.data_ptr() - 8 * self.row_base

    @property
    def succ(self) -> torch.Tensor:
        self.ensure_ready()
        return self.succ_buf

    def ready_slice(self, r0: int, r1: int, ev) -> None:
        """Make rows [r0, r1) of succ valid on `stream` (wait for their upload, relabel)."""
        self.stream.wait_event(ev)
        if self.relabel is not None:
            off, suc, perm, rank = self.relabel
            _lib.check(_lib.hb().hb_relabel_csr_rows(
                self.n, r0, r1, off.data_ptr(), suc.data_ptr(), perm.data_ptr(),
                rank.data_ptr(), self.offsets.data_ptr(), self.succ_buf.data_ptr(),
                self.stream.cuda_stream), "hb_relabel_csr_rows")

    def take_pending(self) -> list:
        """Hand the pending slices to the caller, which must ready_slice() each in order."""
        out, self.pending = self.pending, []
        return out

    def ensure_ready(self) -> None:
        for r0, r1, ev in self.take_pending():
            self.ready_slice(r0, r1, ev)
        self.relabel = None

    @property
    def n_heavy(self) -> int:
        return int(self.heavy_nodes.numel())

    @property
    def n_items(self) -> int:
        return int(self.item_node.numel())

    def to_internal(self, x: torch.Tensor) -> torch.Tensor:
        """Reorder a per-node array from original to internal order."""
        return x if self.perm is None else x.index_select(0, self.perm.long())

    def to_original(self, x: torch.Tensor) -> torch.Tensor:
        return x if self.rank is None else x.index_select(0, self.rank.long())

    def to_internal_bits(self, words: torch.Tensor, n: int) -> torch.Tensor:
        """Change bitmap (int32 words) from original to internal node order."""
        if self.perm is None:
            return words
        return pack_bits(self.to_internal(unpack_bits(words, n)))

    def to_original_bits(self, words: torch.Tensor, n: int) -> torch.Tensor:
        """Change bitmap (int32 words, internal order) -> bool [n] in original order."""
        return self.to_original(unpack_bits(words, n))


def pack_bits(flags: torch.Tensor) -> torch.Tensor:
    """bool [n] -> int32 bitmap [ceil(n/32)], bit v & 31 of word v >> 5."""
    n = flags.numel()
    words = (n + 31) // 32
    padded = torch.zeros(words * 32, dtype=torch.int64, device=flags.device)
    padded[:n] = flags.to(torch.int64)
    shifts = torch.arange(32, dtype=torch.int64, device=flags.device)
    w = (padded.view(words, 32) << shifts).sum(dim=1)
    return torch.where(w >= 2**31, w - 2**32, w).to(torch.int32)


def unpack_bits(words: torch.Tensor, n: int) -> torch.Tensor:
    shifts = torch.arange(32, dtype=torch.int64, device=words.device)
    bits = (words.to(torch.int64).unsqueeze(1) >> shifts) & 1
    return bits.view(-1)[:n].to(torch.bool)


MEGA_ITEMS = 16   # heavy nodes with more work items than this are finished one warp each


_SIDE_STREAMS = {}


def _upload_on_side_stream(a, device, main):
    """int32 successor ids on the device.  A host array is copied on a side stream (the
    copy engine) so that it overlaps the offsets-only work on `main`; returns the tensor
    and the event `main` must wait on (None when nothing was uploaded)."""
    if isinstance(a, torch.Tensor) and a.is_cuda:
        return _as_device(a, torch.int32, device), None
    side = _SIDE_STREAMS.get(device)
    if side is None:
        side = _SIDE_STREAMS[device] = torch.cuda.Stream(device=device)
    side.wait_stream(main)
    with torch.cuda.stream(side):
        t = _as_device(a, torch.int32, device)
        ev = torch.cuda.Event()
        ev.record(side)
    t.record_stream(main)
    return t, ev


# Streamed upload: successor ids of at least STREAM_MIN_ARCS arcs travel in STREAM_SLICES (16:
# config 5 e2e 0.658 -> 0.640 s against 8, config 4 unchanged)
# row slices (one event each), so that the window relabel and iteration 1 run on the
# slices that have arrived while the rest is still crossing PCIe.  HB_STREAM_SLICES=1
# turns it off.
STREAM_SLICES = int(os.environ.get("HB_STREAM_SLICES", "16"))
STREAM_MIN_ARCS = 1 << 24


def slice_rows(off_host: np.ndarray, nslices: int, align: int) -> np.ndarray:
    """Row bounds [0 = r_0 < r_1 < ... = n] of up to `nslices` upload slices holding about
    equal arc counts, every inner bound a multiple of `align` rows (the light kernel's
    chunk window, so the window relabel maps each slice onto itself)."""
    n = off_host.shape[0] - 1
    m = int(off_host[-1])
    targets = np.arange(1, nslices, dtype=np.int64) * m // nslices
    rows = np.searchsorted(off_host, targets, side="left") // align * align
    return np.unique(np.concatenate([[0], rows, [n]])).astype(np.int64)


# Pinned staging buffers for uploads from pageable host memory, per device: two slice
# buffers (int32 ids) and one for the offsets, grown on demand and kept (pinning is slow),
# each with the event of the last copy out of it.
_STAGING = {}
_STAGE_THREADS = int(os.environ.get("HB_STAGE_THREADS", "0"))   # 0 = every core


def _staging(device, key: str, nbytes: int) -> list:
    """[pinned uint8 tensor, event of its last copy] of at least `nbytes` for `device`."""
    pool = _STAGING.setdefault(device, {})
    ent = pool.get(key)
    if ent is None or ent[0].numel() < nbytes:
        if ent is not None and ent[1] is not None:
            ent[1].synchronize()
        ent = pool[key] = [torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True),
                           None]
    return ent


def release_staging_buffers(device=None) -> None:
    """Free the pinned staging buffers kept for uploads from pageable host memory (all
    devices, or one), after their last copies completed.  They are kept between runs
    because pinning is slow; a process that is done uploading large graphs calls this."""
    for dev in list(_STAGING) if device is None else [device]:
        for ent in _STAGING.pop(dev, {}).values():
            if ent[1] is not None:
                ent[1].synchronize()


def _is_pinned(a: np.ndarray) -> bool:
    try:
        with warnings.catch_warnings():   # read-only arrays are only inspected
            warnings.simplefilter("ignore", UserWarning)
            return torch.from_numpy(a[:1]).is_pinned() if a.size else True
    except Exception:
        return False


def _upload_offsets(offsets, device, main) -> torch.Tensor:
    """int64 offsets on the device: a pageable host array is first copied into a pinned
    staging buffer by every core (libhbgraph hbg_stage_bytes), so the DMA runs at the PCIe
    rate instead of through the driver's pageable path."""
    if isinstance(offsets, torch.Tensor):
        return _as_device(offsets, torch.int64, device)
    a = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    if a.size < (1 << 20) or _is_pinned(a):
        return _as_device(a, torch.int64, device)
    ent = _staging(device, "off", a.nbytes)
    if ent[1] is not None:
        ent[1].synchronize()
    _lib.graphlib().hbg_stage_bytes(a.ctypes.data, a.nbytes, ent[0].data_ptr(),
                                    _STAGE_THREADS)
    out = torch.empty(a.shape[0], dtype=torch.int64, device=device)
    with torch.cuda.stream(main):
        out.copy_(ent[0][:a.nbytes].view(torch.int64), non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(main)
    ent[1] = ev
    return out


def _upload_slices(successors, off_host: np.ndarray, device, main, nslices: int, align: int):
    """int32 ids uploaded on the side stream in row slices aligned to `align` rows; returns
    the device tensor and [(r0, r1, event)].  Pinned int32 ids are copied as they are;
    pageable or int64 ids (the reference's CsrGraph) go through two pinned staging
    buffers: every core narrows / copies slice k + 1 into one (hbg_stage_ids) while
    slice k crosses PCIe from the other."""
    n = off_host.shape[0] - 1
    m = int(off_host[-1])
    side = _SIDE_STREAMS.get(device)
    if side is None:
        side = _SIDE_STREAMS[device] = torch.cuda.Stream(device=device)
    side.wait_stream(main)
    dst = torch.empty(m, dtype=torch.int32, device=device)
    arr = np.ascontiguousarray(successors)
    direct = arr.dtype == np.int32 and _is_pinned(arr)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        ht = torch.from_numpy(arr)
    rows = slice_rows(off_host, nslices, align)
    bounds = list(zip(rows[:-1].tolist(), rows[1:].tolist()))
    slices = []
    if direct:
        with torch.cuda.stream(side):
            for r0, r1 in bounds:
                a0, a1 = int(off_host[r0]), int(off_host[r1])
                if a1 > a0:
                    dst[a0:a1].copy_(ht[a0:a1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(side)
                slices.append((r0, r1, ev))
    else:
        G = _lib.graphlib()
        widest = max((int(off_host[r1]) - int(off_host[r0]) for r0, r1 in bounds), default=0)
        bufs = [_staging(device, f"ids{i}", 4 * widest) for i in range(2)]
        for k, (r0, r1) in enumerate(bounds):
            a0, a1 = int(off_host[r0]), int(off_host[r1])
            ent = bufs[k % 2]
            if a1 > a0:
                if ent[1] is not None:
                    ent[1].synchronize()          # its previous slice has left the buffer
                rc = G.hbg_stage_ids(arr.ctypes.data + a0 * arr.itemsize, arr.itemsize,
                                     a1 - a0, ent[0].data_ptr(), _STAGE_THREADS)
                if rc != 0:
                    raise ValueError(f"successor ids of dtype {arr.dtype} are not int32/int64")
                with torch.cuda.stream(side):
                    dst[a0:a1].copy_(ent[0][:4 * (a1 - a0)].view(torch.int32),
                                     non_blocking=True)
            with torch.cuda.stream(side):
                ev = torch.cuda.Event()
                ev.record(side)
            if a1 > a0:
                ent[1] = ev
            slices.append((r0, r1, ev))
    dst.record_stream(side)
    return dst, slices


def _as_device(a, dtype, device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype, non_blocking=True)
    arr = np.ascontiguousarray(a)
    with warnings.catch_warnings():   # read-only host arrays are only copied to the device
        warnings.simplefilter("ignore", UserWarning)
        t = torch.from_numpy(arr)
    return t.to(device=device, non_blocking=True).to(dtype)


# multi-GPU ranks hold only their own rows' successor ids (build_rank_local);
# HB_RANK_LOCAL=0 uploads the whole CSR to every rank (round-1 behaviour)
RANK_LOCAL = bool(int(os.environ.get("HB_RANK_LOCAL", "1")))

WINDOW_MIN_NODES = 1 << 23
# Re-sorting the rows after the degree relabel (hb_sort_rows) makes a hub's consecutive
# arcs read neighbouring register rows: 1-4% off a dense iteration (config 5s 1.80 ->
# 1.74 ms, config 5 38.0 -> 37.5 ms) for a segmented sort of every arc (30 ms at config
# 5s, 0.37 s at config 5) -- a loss for any run of fewer than ~500 iterations.  Off by
# default; HB_SORT_ROWS=1 turns it on.
SORT_ROWS = bool(int(__import__("os").environ.get("HB_SORT_ROWS", "0")))


def choose_order(max_deg: int, light_max_deg: int, n: int = 0) -> str:
    """auto: relabel by degree when any node needs the heavy path (skewed in-degree); else
    sort inside the light kernel's chunks on large graphs (the relabel costs about one
    pass over the CSR, repaid by the dense iterations from ~2^23 nodes: config 4 dense step
    10.98 -> 10.05 ms, run 0.156 -> 0.150 s; config 3 (2^22) step 0.64 -> 0.57 ms but run
    12.8 -> 13.4 ms); identity otherwise."""
    if max_deg > light_max_deg:
        return "degree"
    return "window" if n >= WINDOW_MIN_NODES else "identity"


def _max_degree(off: torch.Tensor, stream) -> int:
    """Largest in-degree of the CSR with device offsets `off` (hb_max_degree)."""
    import ctypes
    n = off.numel() - 1
    if n <= 0:
        return 0
    scratch = torch.empty(1, dtype=torch.int64, device=off.device)
    out = ctypes.c_int64(0)
    _lib.check(_lib.hb().hb_max_degree(n, off.data_ptr(), scratch.data_ptr(), ctypes.byref(out),
                                       stream.cuda_stream), "hb_max_degree")
    return int(out.value)


def node_order(off: torch.Tensor, order: str, b: int, bounds, world: int, stream):
    """(perm, rank, new_offsets) of the `degree` / `window` schedule (hb_schedule_order):
    perm: internal id -> old row; degree: stable sort by descending in-degree, dealt
    round-robin over the ranks (rank r gets ranking positions r, r+W, ...); window: ids
    stay inside the light kernel's grid-stride chunk (aligned as the kernel aligns them per
    rank), sorted by descending in-degree there -- the NPW nodes of a warp round then have
    near-equal in-degrees while id locality (config 4's +-1024 window) is kept.  new_offsets:
    the relabelled CSR's offsets."""
    import ctypes
    n = off.numel() - 1
    dev = off.device
    perm = torch.empty(n, dtype=torch.int32, device=dev)
    rank = torch.empty(n, dtype=torch.int32, device=dev)
    new_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    bnd = np.ascontiguousarray(np.asarray(bounds, dtype=np.int64))
    code = {"degree": 1, "window": 2}[order]
    L = _lib.hb()
    tb = ctypes.c_uint64(0)
    args = (n, off.data_ptr(), code, b, world, bnd.ctypes.data, perm.data_ptr(),
            rank.data_ptr(), new_off.data_ptr())
    _lib.check(L.hb_schedule_order(*args, None, ctypes.byref(tb), stream.cuda_stream),
               "hb_schedule_order(size)")
    temp = torch.empty(max(int(tb.value), 1), dtype=torch.uint8, device=dev)
    _lib.check(L.hb_schedule_order(*args, temp.data_ptr(), ctypes.byref(tb), stream.cuda_stream),
               "hb_schedule_order")
    temp.record_stream(stream)
    return perm, rank, new_off


def heavy_items(row_off: torch.Tensor, nrows: int, lo: int, light_max_deg: int, item_arcs: int,
                stream):
    """Work items of the heavy rows (in-degree > light_max_deg) among rows [lo, lo + nrows)
    whose offsets are row_off[0..nrows] (hb_heavy_items): heavy row ids, item_first,
    item_node, item_beg, finish_order (hubs with more than MEGA_ITEMS items first), n_mega,
    and the number of rows with in-degree > 0."""
    import ctypes
    dev = row_off.device
    L = _lib.hb()
    tb = ctypes.c_uint64(0)
    counts_buf = (ctypes.c_int64 * 4)()
    counts = ctypes.cast(counts_buf, ctypes.c_void_p)
    base = (nrows, lo, row_off.data_ptr(), light_max_deg, item_arcs, MEGA_ITEMS)
    _lib.check(L.hb_heavy_items(*base, None, None, None, None, None, counts, None,
                                ctypes.byref(tb), stream.cuda_stream), "hb_heavy_items(size)")
    temp = torch.empty(max(int(tb.value), 1), dtype=torch.uint8, device=dev)
    _lib.check(L.hb_heavy_items(*base, None, None, None, None, None, counts, temp.data_ptr(),
                                ctypes.byref(tb), stream.cuda_stream), "hb_heavy_items(count)")
    n_heavy, n_items, n_mega, n_nonzero = (int(c) for c in counts_buf)
    heavy = torch.empty(n_heavy, dtype=torch.int32, device=dev)
    item_first = torch.zeros(n_heavy + 1, dtype=torch.int32, device=dev)
    item_node = torch.empty(n_items, dtype=torch.int32, device=dev)
    item_beg = torch.empty(n_items, dtype=torch.int64, device=dev)
    finish_order = torch.empty(n_heavy, dtype=torch.int32, device=dev)
    _lib.check(L.hb_heavy_items(*base, heavy.data_ptr(), item_first.data_ptr(),
                                item_node.data_ptr(), item_beg.data_ptr(),
                                finish_order.data_ptr(), counts, temp.data_ptr(),
                                ctypes.byref(tb), stream.cuda_stream), "hb_heavy_items")
    temp.record_stream(stream)
    return heavy, item_first, n_items, item_node, item_beg, finish_order, n_mega, n_nonzero


def _row_batches(off: torch.Tensor, n: int, m: int, limit: int = (1 << 31) - 1):
    """Row batches of < 2^31 arcs for hb_sort_rows (cub segment sorts take int offsets):
    host arrays of batch start rows and start arcs, found by device searchsorted (no copy
    of the offsets to the host)."""
    rows, arcs = [0], [0]
    while rows[-1] < n:
        a0 = arcs[-1]
        if m - a0 <= limit:
            r1 = n
        else:
            r1 = int(torch.searchsorted(off, torch.tensor([a0 + limit], dtype=off.dtype,
                                                            device=off.device),
                                        right=True).item()) - 1
            r1 = max(r1, rows[-1] + 1)    # a single row above the limit: sorted alone
        rows.append(min(r1, n))
        arcs.append(m if r1 >= n else int(off[r1].item()))
    return np.asarray(rows, dtype=np.int64), np.asarray(arcs, dtype=np.int64)


def partition_bounds(n: int, world: int):
    """Internal-id ranges [bounds[r], bounds[r+1]) owned by each rank (equal node counts;
    in degree order every rank's slice is a round-robin deal of the degree ranking, so
    node and arc counts are balanced together -- SURVEY.md section 8(e))."""
    sizes = [(n - r + world - 1) // world for r in range(world)]   # = len(range(r, n, world))
    bounds = [0]
    for sz in sizes:
        bounds.append(bounds[-1] + sz)
    return bounds


def _upload_owned_rows(ho: np.ndarray, hs: np.ndarray, rows_h: np.ndarray,
                       off_loc_h: np.ndarray, succ: torch.Tensor, rank, device, main) -> None:
    """Successor ids of the owned rows `rows_h` (old row ids, in internal order) into the
    rank-local `succ`, streamed: the rows are cut into up to STREAM_SLICES slices of about
    equal arcs; every host core gathers slice k + 1 (hbg_gather_rows: int32 copy or int64
    narrowing) into one pinned staging buffer while slice k crosses PCIe from the other on
    the side stream, and `main` maps each slice's ids into the internal order
    (hb_map_ids) as it lands."""
    import ctypes
    nloc = rows_h.shape[0]
    mloc = int(off_loc_h[-1]) if nloc else 0
    if mloc == 0:
        return
    nsl = STREAM_SLICES if mloc >= STREAM_MIN_ARCS else 1
    targets = np.arange(1, nsl, dtype=np.int64) * mloc // nsl
    cuts = np.unique(np.concatenate([[0], np.searchsorted(off_loc_h, targets), [nloc]]))
    bounds = [(int(a), int(b)) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
    widest = max(int(off_loc_h[b] - off_loc_h[a]) for a, b in bounds)
    side = _SIDE_STREAMS.get(device)
    if side is None:
        side = _SIDE_STREAMS[device] = torch.cuda.Stream(device=device)
    side.wait_stream(main)
    bufs = [_staging(device, f"rl{i}", 4 * widest) for i in range(2)]
    out_off = np.empty(max(b - a for a, b in bounds) + 1, dtype=np.int64)
    G = _lib.graphlib()
    L = _lib.hb()
    vp = ctypes.c_void_p
    for k, (r0, r1) in enumerate(bounds):
        ent = bufs[k % 2]
        if ent[1] is not None:
            ent[1].synchronize()                # its previous slice has left the buffer
        got = G.hbg_gather_rows(vp(ho.ctypes.data), vp(hs.ctypes.data), hs.itemsize,
                                vp(rows_h.ctypes.data + 4 * r0), r1 - r0, vp(out_off.ctypes.data),
                                vp(ent[0].data_ptr()), 0)
        a0 = int(off_loc_h[r0])
        assert got == int(off_loc_h[r1]) - a0, (got, r0, r1)
        with torch.cuda.stream(side):
            succ[a0:a0 + got].copy_(ent[0][:4 * got].view(torch.int32), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
        ent[1] = ev
        main.wait_event(ev)
        if rank is not None:
            _lib.check(L.hb_map_ids(got, succ.data_ptr() + 4 * a0, rank.data_ptr(),
                                    succ.data_ptr() + 4 * a0, main.cuda_stream), "hb_map_ids")
    succ.record_stream(side)


def build_rank_local(offsets, successors, b: int, device, order: str, world: int,
                     rank_id: int, s_main, on_order=None) -> Schedule:
    """Schedule of one rank of a multi-GPU run with a RANK-LOCAL CSR: the full offsets are
    uploaded (the node order needs every in-degree), but only the successor ids of the
    rows this rank owns -- ~m/W of them -- cross PCIe (gathered on the host by
    hbg_gather_rows into pinned memory), or, for a graph already on the device, are
    gathered there.  Ids are relabelled into the internal order (hashes still use the
    original ids, so registers are bit-identical)."""
    L = _lib.hb()
    off = _upload_offsets(offsets, device, s_main)
    n = off.numel() - 1
    bounds = partition_bounds(n, world)
    lo, hi = bounds[rank_id], bounds[rank_id + 1]
    light_max_deg = int(L.hb_light_max_deg(b))
    item_arcs = int(L.hb_item_arcs(b))
    max_deg = _max_degree(off, s_main)
    if order == "auto":
        order = choose_order(max_deg, light_max_deg, n)
    if order not in ("identity", "degree", "window"):
        raise ValueError(f"unknown schedule order {order!r}")
    perm = rank = None
    new_off = off
    if order in ("degree", "window") and n > 0:
        perm, rank, new_off = node_order(off, order, b, bounds, world, s_main)
    if on_order is not None:
        on_order(perm)
    rows = perm[lo:hi] if perm is not None else torch.arange(lo, hi, dtype=torch.int32,
                                                             device=device)
    nloc = hi - lo
    # offsets of rows [base, hi], base = lo rounded down to 64 rows: the light kernel
    # aligns its warp rounds (and its L2 prefetch of the offsets) below lo; those leading
    # rows are empty here and never valid there.  Positions are local: the owned rows'
    # relabelled offsets minus the first one.
    base = (lo // 64) * 64
    pad = lo - base
    off_pad = torch.zeros(pad + nloc + 1, dtype=torch.int64, device=device)
    off_loc = off_pad[pad:]
    if nloc:
        torch.sub(new_off[lo:hi + 1], new_off[lo], out=off_loc)
    mloc = int(off_loc[-1].item())
    succ = torch.empty(max(mloc, 1), dtype=torch.int32, device=device)
    if isinstance(successors, torch.Tensor) and successors.is_cuda:
        full = successors.to(torch.int32) if successors.dtype != torch.int32 else successors
        ident = torch.arange(n, dtype=torch.int32, device=device) if perm is None else None
        if nloc:
            # k_relabel over new rows [lo, hi): new row i = old row perm[i], ids mapped
            # through rank, written at off_loc[i - lo] (offsets base shifted by lo rows)
            _lib.check(L.hb_relabel_csr_rows(
                n, lo, hi, off.data_ptr(), full.data_ptr(),
                (perm if perm is not None else ident).data_ptr(),
                (rank if rank is not None else ident).data_ptr(),
                off_loc.data_ptr() - 8 * lo, succ.data_ptr(), s_main.cuda_stream),
                "hb_relabel_csr_rows")
    else:
        hs = np.asarray(successors)
        if hs.dtype not in (np.int32, np.int64):
            hs = hs.astype(np.int64)
        hs = np.ascontiguousarray(hs)
        ho = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
        rows_h = np.ascontiguousarray(rows.cpu().numpy().astype(np.int32))
        _upload_owned_rows(ho, hs, rows_h, off_loc.cpu().numpy(), succ, rank, device, s_main)
    heavy, item_first, n_items, item_node, item_beg, finish_order, n_mega, n_nonzero = \
        heavy_items(off_loc, nloc, lo, light_max_deg, item_arcs, s_main)
    p = 1 << b
    # die-affine heavy items (hb_step_args.die_bits) leave two partial rows per item
    partial = torch.empty((max(n_items, 1) * (2 if die_eligible(n, b, order) else 1), p),
                          dtype=torch.uint8, device=device)
    if order == "degree":
        n_heavy = int(heavy.numel())
        light_lo, light_hi = lo + n_heavy, hi
        steady = lo + max(n_nonzero, n_heavy)
    else:
        light_lo, light_hi, steady = lo, hi, hi
    return Schedule(n=n, m=mloc, b=b, order=order, perm=perm, rank=rank, offsets=off_pad,
                    succ_buf=succ[:mloc], lo=lo, hi=hi, light_lo=light_lo, light_hi=light_hi,
                    light_hi_steady=steady, light_max_deg=light_max_deg, item_arcs=item_arcs,
                    heavy_nodes=heavy, item_first=item_first,
                    finish_order=finish_order, n_mega=n_mega,
                    item_node=item_node, item_beg=item_beg,
                    partial=partial, max_deg=max_deg,
                    hot_rows=hot_head_rows(n, order, world), stream=s_main, row_base=base,
                    local=True)


def build_schedule(offsets, successors, b: int, device, order: str = "auto", world: int = 1,
                   rank_id: int = 0, stream=None, on_order=None) -> Schedule:
    """Upload the CSR of G^T, relabel it into schedule order and split the heavy nodes of
    this rank's internal-id range [lo, hi) into work items.

    The successor ids (the bulk of the upload) travel on a side stream while the offsets-
    only work runs (degrees, node order); on_order(perm), if given, is called once the
    order is known and before the ids are needed, so the caller can launch work that
    overlaps the rest of the upload (the engine seeds the counters there)."""
    L = _lib.hb()
    s_main = stream if stream is not None else torch.cuda.current_stream(device)
    if world > 1 and RANK_LOCAL:
        return build_rank_local(offsets, successors, b, device, order, world, rank_id,
                                s_main, on_order)
    off = _upload_offsets(offsets, device, s_main)
    slices = None
    if (world == 1 and STREAM_SLICES > 1 and not isinstance(successors, torch.Tensor)
            and not isinstance(offsets, torch.Tensor)
            and np.asarray(successors).dtype in (np.int32, np.int64)
            and np.asarray(successors).shape[0] >= STREAM_MIN_ARCS):
        off_host = np.asarray(offsets, dtype=np.int64)
        succ, slices = _upload_slices(successors, off_host, device, s_main, STREAM_SLICES,
                                      int(L.hb_light_window(b)))
        ids_ready = None
    else:
        succ, ids_ready = _upload_on_side_stream(successors, device, s_main)
    n = off.numel() - 1
    m = succ.numel()
    bounds = partition_bounds(n, world)
    lo, hi = bounds[rank_id], bounds[rank_id + 1]
    light_max_deg = int(L.hb_light_max_deg(b))
    item_arcs = int(L.hb_item_arcs(b))
    max_deg = _max_degree(off, s_main)
    if order == "auto":
        order = choose_order(max_deg, light_max_deg, n)
    if order not in ("identity", "degree", "window"):
        raise ValueError(f"unknown schedule order {order!r}")
    perm = rank = new_off = None
    if order in ("window", "degree") and n > 0:
        # perm, its inverse and the relabelled offsets, on the device (hb_schedule_order)
        perm, rank, new_off = node_order(off, order, b, bounds, world, s_main)
    if on_order is not None:
        on_order(perm)
    if ids_ready is not None:
        s_main.wait_event(ids_ready)
    pending, relabel, src_slices, late_relabel = [], None, None, None
    if slices is not None:
        if order in ("window", "identity") and n > 0:
            pending = slices                   # consumed by iteration 1, slice by slice
        elif order == "degree" and n > 0:
            src_slices = slices                # relabelled slice by slice as they land
        else:
            for _, _, ev in slices:
                s_main.wait_event(ev)
    if order == "window" and n > 0 and pending:
        relabel = (off, succ, perm, rank)      # window slices map onto themselves
        off, succ = new_off, torch.empty(m, dtype=torch.int32, device=device)
    elif order == "window" and n > 0:
        new_succ = torch.empty(m, dtype=torch.int32, device=device)
        s = s_main
        _lib.check(L.hb_relabel_csr(n, off.data_ptr(), succ.data_ptr(), perm.data_ptr(),
                                    rank.data_ptr(), new_off.data_ptr(), new_succ.data_ptr(),
                                    s.cuda_stream), "hb_relabel_csr")
        # ids move by less than a window: rows stay nearly ascending, no re-sort needed
        off, succ = new_off, new_succ
    if order == "degree" and n > 0:
        new_succ = torch.empty(m, dtype=torch.int32, device=device)
        s = s_main
        if src_slices is not None and not SORT_ROWS:
            # scatter form by uploaded (old) rows: slice k is relabelled while slices
            # k+1.. are still crossing PCIe; every new row is complete after the last one.
            # Enqueued at the end, after the heavy-item setup below, whose host reads must
            # not wait for the copy.
            def late_relabel(off=off, succ=succ, rank=rank, new_off=new_off,
                             new_succ=new_succ, s=s):
                for r0, r1, ev in src_slices:
                    s.wait_event(ev)
                    _lib.check(L.hb_relabel_csr_src_rows(
                        n, r0, r1, off.data_ptr(), succ.data_ptr(), rank.data_ptr(),
                        new_off.data_ptr(), new_succ.data_ptr(), s.cuda_stream),
                        "hb_relabel_csr_src_rows")
        elif src_slices is not None:
            for _, _, ev in src_slices:
                s.wait_event(ev)
            _lib.check(L.hb_relabel_csr(n, off.data_ptr(), succ.data_ptr(), perm.data_ptr(),
                                        rank.data_ptr(), new_off.data_ptr(),
                                        new_succ.data_ptr(), s.cuda_stream), "hb_relabel_csr")
        else:
            _lib.check(L.hb_relabel_csr(n, off.data_ptr(), succ.data_ptr(), perm.data_ptr(),
                                        rank.data_ptr(), new_off.data_ptr(),
                                        new_succ.data_ptr(), s.cuda_stream), "hb_relabel_csr")
        # optionally restore ascending ids inside every row (graph.py's normalisation), in
        # internal ids: a hub's consecutive arcs then read neighbouring register rows
        if SORT_ROWS:
            brows, barcs = _row_batches(new_off, n, m)
            if isinstance(successors, torch.Tensor) and successors.data_ptr() == succ.data_ptr():
                succ = torch.empty_like(succ)       # never scribble on the caller's tensor
            import ctypes
            tb = ctypes.c_uint64(0)
            br = brows.ctypes.data_as(ctypes.c_void_p)
            ba = barcs.ctypes.data_as(ctypes.c_void_p)
            nb = brows.size - 1
            _lib.check(L.hb_sort_rows(n, new_off.data_ptr(), nb, br, ba, new_succ.data_ptr(),
                                      succ.data_ptr(), None, ctypes.byref(tb), None,
                                      s.cuda_stream), "hb_sort_rows(size)")
            temp = torch.empty(max(int(tb.value), 1), dtype=torch.uint8, device=device)
            _lib.check(L.hb_sort_rows(n, new_off.data_ptr(), nb, br, ba, new_succ.data_ptr(),
                                      succ.data_ptr(), temp.data_ptr(), ctypes.byref(tb), None,
                                      s.cuda_stream), "hb_sort_rows")
            del temp
        off, succ = new_off, new_succ
    # heavy rows of [lo, hi) and their work items, on the device (hb_heavy_items)
    heavy, item_first, n_items, item_node, item_beg, finish_order, n_mega, n_nonzero = \
        heavy_items(off[lo:], hi - lo, lo, light_max_deg, item_arcs, s_main)
    p = 1 << b
    # die-affine heavy items (hb_step_args.die_bits) leave two partial rows per item
    partial = torch.empty((max(n_items, 1) * (2 if die_eligible(n, b, order) else 1), p),
                          dtype=torch.uint8, device=device)
    if order == "degree":
        # this rank's slice is in descending degree: heavy first, zero in-degree last
        n_heavy = int(heavy.numel())
        light_lo, light_hi = lo + n_heavy, hi
        steady = lo + max(n_nonzero, n_heavy)
    else:
        light_lo, light_hi, steady = lo, hi, hi
    if late_relabel is not None:
        late_relabel()
    return Schedule(n=n, m=m, b=b, order=order, perm=perm, rank=rank, offsets=off, succ_buf=succ,
                    lo=lo, hi=hi, light_lo=light_lo, light_hi=light_hi,
                    light_hi_steady=steady, light_max_deg=light_max_deg, item_arcs=item_arcs,
                    heavy_nodes=heavy, item_first=item_first,
                    finish_order=finish_order, n_mega=n_mega,
                    item_node=item_node, item_beg=item_beg,
                    partial=partial, max_deg=max_deg,
                    hot_rows=hot_head_rows(n, order, world), pending=pending,
                    relabel=relabel, stream=s_main)
