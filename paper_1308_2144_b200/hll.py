"""Counter parameters, host-side hashing and the at-rest packed counter format.

Same public names, argument meanings and errors as the reference's ``hll.py``; the
bodies are independent restatements (the device does the real hashing in ``k_seed``):

* ``CounterParams``                       hll.py:109-144
* ``alpha`` / ``POW2NEG``                 hll.py:33,40-48
* ``hash_items`` / ``hash_item``          hll.py:70-95
* ``register_values``                     hll.py:147-158
* ``pack_rows`` / ``unpack_rows``         hll.py:161-177 (width-bit fields, MSB first)
* ``CounterArray``                        hll.py:180-319 (representation + ``HLLA`` blob)

New here: ``estimator_constants`` (engine.py:149-151 evaluated in the same order) and
``lc_table``, the linear-counting values ``p * ln(p / V)`` built with ``math.log``
(bit-identical to numba's ``np.log`` in ``_kernels.py:33``)
that the device estimator reads instead of evaluating a CUDA ``log``.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass

import numpy as np

BLOB_MAGIC = b"HLLA"
BLOB_VERSION = 1
_MASK64 = (1 << 64) - 1
_BLOB_HEADER = struct.Struct("<HBBQQ")   # version, b, width, n, seed

# 2^-r for every byte value r (exact powers of two)
POW2NEG = np.ldexp(1.0, -np.arange(256)).astype(np.float64)


class BlobFormatError(ValueError):
    """Raised when a serialized counter-array blob is malformed."""


def alpha(p: int) -> float:
    """HLL bias constant alpha_p: tabulated for p in {16, 32, 64}, closed form above."""
    table = {16: 0.673, 32: 0.697, 64: 0.709}
    if p in table:
        return table[p]
    return 0.7213 / (1.0 + 1.079 / p)


def standard_deviation_bound(p: int) -> float:
    if p < 16:
        raise ValueError(f"p must be >= 16, got {p}")
    return 1.06 / math.sqrt(p)


def estimator_constants(p: int):
    """(alpha_p2, lc_cut, p_float); alpha_p2 multiplies left to right like the reference."""
    a = alpha(p)
    return (a * p) * p, 2.5 * p, float(p)


def lc_table(p: int) -> np.ndarray:
    """lc[V] = float(p) * math.log(float(p) / V) for V in 1..p; lc[0] is unused."""
    pf = float(p)
    return np.array([0.0] + [pf * math.log(pf / v) for v in range(1, p + 1)],
                    dtype=np.float64)


_FINALIZER = ((30, 0xBF58476D1CE4E5B9), (27, 0x94D049BB133111EB))


def _splitmix_finalize(z: np.ndarray) -> np.ndarray:
    """splitmix64 output finaliser over a uint64 array, wrapping mod 2^64."""
    with np.errstate(over="ignore"):
        for shift, mult in _FINALIZER:
            z = (z ^ (z >> np.uint64(shift))) * np.uint64(mult)
        return z ^ (z >> np.uint64(31))


def hash_items(items, replicas, seed: int) -> np.ndarray:
    """h = F(item + F(replica + F(seed))) with F the splitmix64 finaliser (wrapping)."""
    it = np.atleast_1d(np.asarray(items, dtype=np.uint64))
    rp = np.atleast_1d(np.asarray(replicas, dtype=np.uint64))
    s = _splitmix_finalize(np.array([seed & _MASK64], dtype=np.uint64))
    with np.errstate(over="ignore"):
        keyed = _splitmix_finalize(rp + s)
        return _splitmix_finalize(it + keyed)


def hash_item(item: int, replica: int = 0, seed: int = 0) -> int:
    return int(hash_items([item], [replica], seed)[0])


def _bit_length(x: np.ndarray) -> np.ndarray:
    """Exact bit length of uint64 values via frexp on the two 32-bit halves."""
    hi = (x >> np.uint64(32)).astype(np.float64)
    lo = (x & np.uint64(0xFFFFFFFF)).astype(np.float64)
    bl_hi = np.frexp(hi)[1].astype(np.int64)
    bl_lo = np.frexp(lo)[1].astype(np.int64)
    return np.where(hi > 0, 32 + bl_hi, bl_lo)


@dataclass(frozen=True)
class CounterParams:
    """p = 2^b registers of register_width bits each, hashed under `seed`."""

    b: int
    register_width: int = 5
    seed: int = 0

    def __post_init__(self) -> None:
        if self.b < 4:
            raise ValueError(f"b must be >= 4 (p >= 16), got {self.b}")
        if self.register_width < 1 or self.register_width > 8:
            raise ValueError(
                f"register_width must be in [1, 8], got {self.register_width}")

    @property
    def p(self) -> int:
        return 2 ** self.b

    @property
    def row_bytes(self) -> int:
        return (self.p * self.register_width) // 8

    @property
    def saturation(self) -> int:
        return 2 ** self.register_width - 1

    @property
    def rho_max(self) -> int:
        return 65 - self.b

    def rsd_bound(self) -> float:
        return standard_deviation_bound(self.p)


def register_values(hashes, params: CounterParams):
    """(register index, rho) per hash: low b bits pick the register; rho is one plus the
    leading-zero count of the remaining 64-b bits, clamped to the saturation value."""
    h = np.asarray(hashes, dtype=np.uint64)
    idx = (h % np.uint64(params.p)).astype(np.int64)
    rho = params.rho_max - _bit_length(h >> np.uint64(params.b))
    return idx, np.minimum(rho, params.saturation).astype(np.uint8)


def pack_rows(dense: np.ndarray, register_width: int) -> np.ndarray:
    """(k, p) byte registers -> (k, p*width/8) bytes, each register's `width` low bits
    written most-significant first, rows concatenated without padding."""
    d = np.ascontiguousarray(dense, dtype=np.uint8)
    k, p = d.shape
    bits8 = np.unpackbits(d.reshape(k, p, 1), axis=2)          # MSB-first, 8 per register
    fields = bits8[:, :, 8 - register_width:].reshape(k, p * register_width)
    return np.packbits(fields, axis=1)


def unpack_rows(packed: np.ndarray, p: int, register_width: int) -> np.ndarray:
    pk = np.atleast_2d(np.asarray(packed, dtype=np.uint8))
    k = pk.shape[0]
    fields = np.unpackbits(pk, axis=1)[:, :p * register_width].reshape(k, p, register_width)
    bits8 = np.zeros((k, p, 8), dtype=np.uint8)
    bits8[:, :, 8 - register_width:] = fields
    return np.packbits(bits8, axis=2).reshape(k, p)


class CounterArray:
    """n packed counters sharing one CounterParams: the at-rest form of the registers."""

    def __init__(self, n: int, params: CounterParams, registers: np.ndarray | None = None):
        if n < 0:
            raise ValueError("n must be non-negative")
        shape = (n, params.row_bytes)
        regs = (np.zeros(shape, dtype=np.uint8) if registers is None
                else np.asarray(registers, dtype=np.uint8))
        if regs.shape != shape:
            raise ValueError(
                f"registers shape {regs.shape} does not match (n={n}, "
                f"row_bytes={params.row_bytes})")
        self.n, self.params, self.registers = n, params, regs

    @property
    def nbytes(self) -> int:
        return self.registers.nbytes

    @classmethod
    def from_dense(cls, dense, params: CounterParams) -> "CounterArray":
        d = np.atleast_2d(np.asarray(dense, dtype=np.uint8))
        if d.shape[1] != params.p:
            raise ValueError("dense register matrix has wrong register count")
        if d.size and int(d.max()) > params.saturation:
            raise ValueError("register value exceeds saturation for this width")
        return cls(d.shape[0], params, pack_rows(d, params.register_width))

    def to_dense(self, rows=None) -> np.ndarray:
        sel = self.registers if rows is None else self.registers[rows]
        if len(sel) == 0:
            return np.zeros((0, self.params.p), dtype=np.uint8)
        return unpack_rows(sel, self.params.p, self.params.register_width)

    def copy(self) -> "CounterArray":
        return CounterArray(self.n, self.params, self.registers.copy())

    def __eq__(self, other) -> bool:
        if not isinstance(other, CounterArray):
            return NotImplemented
        return (self.n, self.params) == (other.n, other.params) and bool(
            np.array_equal(self.registers, other.registers))

    def to_blob(self) -> bytes:
        pr = self.params
        head = _BLOB_HEADER.pack(BLOB_VERSION, pr.b, pr.register_width, self.n,
                                 pr.seed & _MASK64)
        return BLOB_MAGIC + head + self.registers.tobytes()

    @classmethod
    def from_blob(cls, blob: bytes) -> "CounterArray":
        hdr = 4 + _BLOB_HEADER.size
        if len(blob) < hdr or blob[:4] != BLOB_MAGIC:
            raise BlobFormatError("bad counter-array magic")
        version, b, width, n, seed = _BLOB_HEADER.unpack_from(blob, 4)
        if version != BLOB_VERSION:
            raise BlobFormatError(f"unsupported blob version {version}")
        params = CounterParams(b=b, register_width=width, seed=seed)
        if len(blob) != hdr + n * params.row_bytes:
            raise BlobFormatError(
                f"blob length {len(blob)} != expected {hdr + n * params.row_bytes}")
        regs = np.frombuffer(blob, dtype=np.uint8, offset=hdr).reshape(n, params.row_bytes)
        return cls(n, params, regs.copy())
