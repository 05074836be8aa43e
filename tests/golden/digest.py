"""Chunked register digest shared by make_fullsize.py (reference side) and
tests/test_gpu_fullsize.py (device side)."""

import hashlib
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

CHUNK = 64 << 20


def reg_digest(a: np.ndarray, threads: int | None = None) -> str:
    """sha256 over the sha256 digests of consecutive 64 MiB chunks of the C-order bytes
    (the chunks hash in parallel: a 4.3 GB register matrix takes about a second)."""
    buf = memoryview(np.ascontiguousarray(a)).cast("B")
    chunks = [buf[i:i + CHUNK] for i in range(0, len(buf), CHUNK)] or [buf]
    with ThreadPoolExecutor(threads or os.cpu_count() or 1) as ex:
        parts = list(ex.map(lambda c: hashlib.sha256(c).digest(), chunks))
    return hashlib.sha256(b"".join(parts)).hexdigest()
