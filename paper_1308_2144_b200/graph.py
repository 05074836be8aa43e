"""Host-side CSR graphs: the input boundary of the hot path.

``CsrGraph`` keeps the reference's interface (graph.py:29-97: ``n``, ``m``,
``offsets``, ``successors``, ``successors_of``, ``out_degrees``, ``from_edges``) and its
normalisation (sorted successor lists, duplicates removed), but stores successor ids as
int32 whenever n fits -- the device consumes int32 ids, and a 4-byte id halves the CSR
traffic of the union kernel.  Any object with ``offsets``/``successors``
arrays (e.g. the reference's own ``hyperball.CsrGraph``) is accepted by the engine.

``transpose`` (graph.py:145-155) and the ``CSR1`` binary format (graph.py:158-215:
magic, n u64, m u64, (n+1) u64 offsets, m u64 successors) are restated here so graphs
can be exchanged with the reference CLI.
"""

from __future__ import annotations

import struct
import warnings
from pathlib import Path

import numpy as np

BINARY_MAGIC = b"CSR1"
HEADER_BYTES = 20


class GraphFormatError(ValueError):
    """Malformed binary graph file."""


def _id_dtype(n: int):
    return np.int32 if n < 2**31 else np.int64


class CsrGraph:
    """Immutable CSR: offsets int64 [n+1], successors int32/int64 [m]."""

    __slots__ = ("n", "m", "offsets", "successors", "__weakref__")

    def __init__(self, offsets, successors):
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        if off.ndim != 1 or off.size < 1:
            raise ValueError("offsets must be a 1-d array of length n + 1")
        n = off.size - 1
        suc = np.ascontiguousarray(successors)
        if suc.dtype not in (np.int32, np.int64):
            suc = suc.astype(np.int64)
        if suc.dtype == np.int64 and n < 2**31:
            suc = suc.astype(np.int32)
        m = suc.size
        if off[0] != 0 or off[-1] != m or (n and bool((off[1:] < off[:-1]).any())):
            raise ValueError("offsets must grow monotonically from 0 to m")
        if m and (int(suc.min()) < 0 or int(suc.max()) >= n):
            raise ValueError("successor id out of range")
        off.setflags(write=False)
        suc.setflags(write=False)
        self.n, self.m, self.offsets, self.successors = n, m, off, suc

    @classmethod
    def from_edges(cls, src, dst, n: int | None = None) -> "CsrGraph":
        """Normalised graph (sorted, deduplicated successor lists) from arc arrays."""
        s = np.asarray(src, dtype=np.int64).ravel()
        d = np.asarray(dst, dtype=np.int64).ravel()
        if s.shape != d.shape:
            raise ValueError("src and dst must have equal length")
        if s.size and min(int(s.min()), int(d.min())) < 0:
            raise ValueError("node ids must be non-negative")
        top = int(max(s.max(), d.max())) + 1 if s.size else 0
        if n is None:
            n = top
        elif top > n:
            raise ValueError(f"node id {top - 1} >= declared node count {n}")
        key = np.unique(s * max(n, 1) + d)               # sorted by (src, dst), deduplicated
        s, d = key // max(n, 1), key % max(n, 1)
        offsets = np.zeros(n + 1, dtype=np.int64)
        offsets[1:] = np.cumsum(np.bincount(s, minlength=n))
        return cls(offsets, d.astype(_id_dtype(n)))

    def successors_of(self, v: int) -> np.ndarray:
        return self.successors[self.offsets[v]:self.offsets[v + 1]]

    @property
    def out_degrees(self) -> np.ndarray:
        return np.diff(self.offsets)

    def __eq__(self, other) -> bool:
        if not hasattr(other, "offsets") or not hasattr(other, "successors"):
            return NotImplemented
        return (self.n == other.n and self.m == other.m
                and np.array_equal(self.offsets, other.offsets)
                and np.array_equal(self.successors, other.successors))

    def __repr__(self) -> str:
        return f"CsrGraph(n={self.n}, m={self.m})"


class DeviceCsrGraph:
    """A CSR already resident on a CUDA device (offsets int64 [n+1], successors int32 [m]
    torch tensors), e.g. from the GPU graph builders; accepted wherever a CsrGraph is."""

    __slots__ = ("n", "m", "offsets", "successors", "__weakref__")

    def __init__(self, offsets, successors):
        self.offsets, self.successors = offsets, successors
        self.n = int(offsets.numel()) - 1
        self.m = int(successors.numel())

    def to_host(self) -> CsrGraph:
        return CsrGraph(self.offsets.cpu().numpy(), self.successors.cpu().numpy())

    def __repr__(self) -> str:
        return f"DeviceCsrGraph(n={self.n}, m={self.m}, device={self.offsets.device})"


def transpose_device(g, device=None) -> DeviceCsrGraph:
    """transpose (graph.py:145-155) on the GPU: every arc reversed, duplicates and
    self-loops kept, each new row listing its sources in ascending order -- the
    reference's stable argsort by target, as one radix sort of (target << 32 | source)
    keys (hb_transpose_csr).  Accepts a host or device CSR; returns a DeviceCsrGraph."""
    import ctypes

    import torch

    from ._lib import check, hb
    if isinstance(g.offsets, torch.Tensor) and g.offsets.is_cuda:
        dev = g.offsets.device
    else:
        dev = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
    with torch.cuda.device(dev):
        def up(a, dt):
            if isinstance(a, torch.Tensor):
                return a.to(device=dev, dtype=dt).contiguous()
            with warnings.catch_warnings():      # read-only host arrays are only copied
                warnings.simplefilter("ignore", UserWarning)
                return torch.from_numpy(np.ascontiguousarray(a)).to(dev).to(dt)
        off = up(g.offsets, torch.int64)
        suc = up(g.successors, torch.int32)
        n, m = off.numel() - 1, suc.numel()
        stream = torch.cuda.current_stream(dev)
        keys = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
        alt = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
        tb = ctypes.c_uint64(0)
        L = hb()
        check(L.hb_transpose_csr(n, m, off.data_ptr(), suc.data_ptr(), keys.data_ptr(),
                                 alt.data_ptr(), None, ctypes.byref(tb), None, None,
                                 stream.cuda_stream), "hb_transpose_csr(size)")
        temp = torch.empty(max(int(tb.value), 1), dtype=torch.uint8, device=dev)
        out_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
        out_suc = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
        check(L.hb_transpose_csr(n, m, off.data_ptr(), suc.data_ptr(), keys.data_ptr(),
                                 alt.data_ptr(), temp.data_ptr(), ctypes.byref(tb),
                                 out_off.data_ptr(), out_suc.data_ptr(), stream.cuda_stream),
              "hb_transpose_csr")
        del keys, alt, temp
    return DeviceCsrGraph(out_off, out_suc[:m])


def transpose(g) -> CsrGraph:
    """Reverse every arc; the result is normalised (sorted rows).  A DeviceCsrGraph is
    transposed on its device (transpose_device)."""
    if isinstance(g, DeviceCsrGraph):
        return transpose_device(g)
    n = int(np.asarray(g.offsets).size - 1)
    deg = np.diff(np.asarray(g.offsets, dtype=np.int64))
    src = np.repeat(np.arange(n, dtype=np.int64), deg)
    dst = np.asarray(g.successors, dtype=np.int64)
    order = np.lexsort((src, dst))                      # by new row, then new successor
    offsets = np.zeros(n + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(np.bincount(dst, minlength=n))
    return CsrGraph(offsets, src[order].astype(_id_dtype(n)))


def write_binary(g, sink) -> None:
    if isinstance(sink, (str, Path)):
        with open(sink, "wb") as fh:
            write_binary(g, fh)
        return
    n = int(np.asarray(g.offsets).size - 1)
    sink.write(BINARY_MAGIC + struct.pack("<QQ", n, int(np.asarray(g.successors).size)))
    sink.write(np.asarray(g.offsets, dtype="<u8").tobytes())
    sink.write(np.asarray(g.successors, dtype="<u8").tobytes())


def read_binary(source, mmap: bool = False) -> CsrGraph:
    if isinstance(source, (str, Path)):
        path = Path(source)
        if mmap:
            with open(path, "rb") as fh:
                head = fh.read(HEADER_BYTES)
            n, m = _check_header(head, path.stat().st_size)
            off = np.memmap(path, dtype="<u8", mode="r", offset=HEADER_BYTES, shape=(n + 1,))
            suc = np.memmap(path, dtype="<u8", mode="r", offset=HEADER_BYTES + 8 * (n + 1),
                            shape=(m,))
            return _make(off.view(np.int64), suc.view(np.int64))
        with open(path, "rb") as fh:
            return read_binary(fh)
    data = source.read()
    n, m = _check_header(data[:HEADER_BYTES], len(data))
    off = np.frombuffer(data, dtype="<u8", count=n + 1, offset=HEADER_BYTES)
    suc = np.frombuffer(data, dtype="<u8", count=m, offset=HEADER_BYTES + 8 * (n + 1))
    return _make(off.astype(np.int64), suc.astype(np.int64))


def _check_header(head: bytes, size: int):
    if len(head) < HEADER_BYTES or head[:4] != BINARY_MAGIC:
        raise GraphFormatError("bad graph magic")
    n, m = struct.unpack("<QQ", head[4:HEADER_BYTES])
    if size != HEADER_BYTES + 8 * (n + 1) + 8 * m:
        raise GraphFormatError(
            f"file length {size} != expected {HEADER_BYTES + 8 * (n + 1) + 8 * m} "
            f"for n={n}, m={m}")
    return n, m


def _make(off, suc) -> CsrGraph:
    try:
        return CsrGraph(off, suc)
    except ValueError as exc:
        raise GraphFormatError(str(exc)) from None
