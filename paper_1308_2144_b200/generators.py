"""Synthetic graphs of the five BASELINE.json configs (SURVEY.md Appendix B,
BASELINE.md section 4), built by the host C library ``libhbgraph.so``.

Every builder returns the CSR of the TRANSPOSE graph G^T -- the graph the engine runs
on for the default ``--direction negative`` (cli.py:213-216) -- with self-loops dropped
and duplicate arcs removed.  Randomness is counter-based, so a config is a pure function
of its parameters: the GPU run, the CPU oracle and the golden fixtures all see the same
bytes (tests pin the digests).

Pinned choices: hash seed 42 for every config, register
width 5, config 4's Zipf(2.1) out-degree on {3..10^4} (mean 15.7; BASELINE.md section 4
explains why), R-MAT without noise or label permutation.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
from dataclasses import dataclass

import numpy as np

from ._lib import graphlib
from .graph import CsrGraph

RMAT_ABC = (0.57, 0.19, 0.19)


def _threads(threads: int | None) -> int:
    return int(threads) if threads else (os.cpu_count() or 1)


def _collect(handle) -> CsrGraph:
    L = graphlib()
    try:
        n, m = L.hbg_n(handle), L.hbg_m(handle)
        off = np.empty(n + 1, dtype=np.int64)
        suc = np.empty(m, dtype=np.int32)
        L.hbg_copy(handle, off.ctypes.data_as(ctypes.c_void_p), suc.ctypes.data_as(ctypes.c_void_p))
    finally:
        L.hbg_free(handle)
    return CsrGraph(off, suc)


def erdos_renyi_t(n: int, mean_degree: float, seed: int, threads: int | None = None) -> CsrGraph:
    """Directed ER: out-degree Poisson(mean), targets uniform on V minus the source."""
    return _collect(graphlib().hbg_er(n, float(mean_degree), seed, _threads(threads)))


def rmat_t(scale: int, arcs: int, seed: int, abc=RMAT_ABC, threads: int | None = None) -> CsrGraph:
    """R-MAT with `arcs` generated arcs on 2^scale nodes (before dedup / self-loop removal)."""
    a, b, c = abc
    return _collect(graphlib().hbg_rmat(scale, arcs, a, b, c, seed, _threads(threads)))


def rmat_t_device(scale: int, arcs: int, seed: int, abc=RMAT_ABC, device=None):
    """rmat_t built on the GPU (hb_gen_rmat_keys + hb_keys_to_csr): the same bytes as the
    host builder (tests pin the digest), as a DeviceCsrGraph.  Peak device memory is about
    20 bytes per generated arc."""
    import torch

    from ._lib import check, hb
    from .graph import DeviceCsrGraph

    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    a, b, c = abc
    thr = [int(a * 4294967296.0), int((a + b) * 4294967296.0), int((a + b + c) * 4294967296.0)]
    n = 1 << scale
    L = hb()
    stream = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        keys = torch.empty(arcs, dtype=torch.int64, device=dev)
        alt = torch.empty(arcs, dtype=torch.int64, device=dev)
        check(L.hb_gen_rmat_keys(scale, arcs, thr[0], thr[1], thr[2], seed, keys.data_ptr(),
                                 stream.cuda_stream), "hb_gen_rmat_keys")
        tb = ctypes.c_uint64(0)
        mo = ctypes.c_int64(0)
        check(L.hb_keys_to_csr(n, arcs, keys.data_ptr(), alt.data_ptr(), None, ctypes.byref(tb),
                               ctypes.byref(mo), None, None, stream.cuda_stream), "size")
        temp = torch.empty(int(tb.value), dtype=torch.uint8, device=dev)
        offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
        succ = torch.empty(arcs, dtype=torch.int32, device=dev)
        check(L.hb_keys_to_csr(n, arcs, keys.data_ptr(), alt.data_ptr(), temp.data_ptr(),
                               ctypes.byref(tb), ctypes.byref(mo), offsets.data_ptr(),
                               succ.data_ptr(), stream.cuda_stream), "hb_keys_to_csr")
        del keys, alt, temp
        succ = succ[:mo.value].clone()
    return DeviceCsrGraph(offsets, succ)


def disconnected_t(n: int, giant: int, geo_p: float, mean_degree: float, seed: int,
                   threads: int | None = None) -> CsrGraph:
    """Giant block [0, giant) plus consecutive Geometric(geo_p)-sized blocks; each node
    draws Poisson(mean) out-arcs to uniform targets inside its own block."""
    return _collect(graphlib().hbg_disconnected(n, giant, geo_p, float(mean_degree), seed,
                                                _threads(threads)))


def weblike_t(n: int, seed: int, alpha: float = 2.1, kmin: int = 3, kmax: int = 10_000,
              p_local: float = 0.8, window: int = 1024, threads: int | None = None) -> CsrGraph:
    """Zipf(alpha) out-degree on {kmin..kmax}; an arc is local (u +- U{1..window} mod n)
    with probability p_local, else uniform."""
    return _collect(graphlib().hbg_weblike(n, alpha, kmin, kmax, p_local, window, seed,
                                           _threads(threads)))


def from_arcs_t(n: int, src, dst, threads: int | None = None) -> CsrGraph:
    """G^T of an explicit arc list (self-loops dropped, deduplicated, rows sorted)."""
    s = np.ascontiguousarray(src, dtype=np.uint32)
    d = np.ascontiguousarray(dst, dtype=np.uint32)
    h = graphlib().hbg_from_arcs(n, s.size, s.ctypes.data_as(ctypes.c_void_p),
                                 d.ctypes.data_as(ctypes.c_void_p), _threads(threads))
    return _collect(h)


@dataclass(frozen=True)
class BenchConfig:
    name: str
    log2m: int
    hash_seed: int
    outputs: tuple
    description: str

    def build(self, threads: int | None = None) -> CsrGraph:
        return BUILDERS[self.name](threads)

    def build_device(self, device=None):
        """GPU-built graph where a device builder exists (R-MAT configs), else the host
        graph (the engine uploads it)."""
        if self.name in DEVICE_BUILDERS:
            return DEVICE_BUILDERS[self.name](device)
        return self.build()


BUILDERS = {
    "config1": lambda th=None: erdos_renyi_t(10_000, 8.0, seed=0, threads=th),
    "config2": lambda th=None: rmat_t(20, 16 << 20, seed=1, threads=th),
    "config3": lambda th=None: disconnected_t(1 << 22, 1 << 21, 0.1, 6.0, seed=2, threads=th),
    "config4": lambda th=None: weblike_t(1 << 24, seed=3, threads=th),
    "config5": lambda th=None: rmat_t(28, 1 << 32, seed=4, threads=th),
    # config 5 at 1/16 scale (same law, same parameters): for iteration on smaller boxes
    "config5s": lambda th=None: rmat_t(24, 1 << 28, seed=4, threads=th),
}

DEVICE_BUILDERS = {
    "config2": lambda dev=None: rmat_t_device(20, 16 << 20, seed=1, device=dev),
    "config5": lambda dev=None: rmat_t_device(28, 1 << 32, seed=4, device=dev),
    "config5s": lambda dev=None: rmat_t_device(24, 1 << 28, seed=4, device=dev),
}

CONFIGS = {
    "config1": BenchConfig("config1", 6, 42, ("harmonic", "closeness", "lin"),
                           "ER n=10^4, out-degree Poisson(8), seed 0, log2m 6"),
    "config2": BenchConfig("config2", 7, 42, ("harmonic", "closeness", "lin"),
                           "R-MAT scale 20, 16*2^20 arcs, (.57,.19,.19,.05), seed 1, log2m 7"),
    "config3": BenchConfig("config3", 6, 42, ("harmonic", "closeness", "lin"),
                           "n=2^22: giant 2^21 + Geometric(0.1) blocks, Poisson(6), seed 2, log2m 6"),
    "config4": BenchConfig("config4", 8, 42, ("harmonic", "closeness", "lin"),
                           "web-like n=2^24, Zipf(2.1) on {3..10^4}, 80% within +-1024, seed 3, log2m 8"),
    "config5": BenchConfig("config5", 4, 42, ("harmonic",),
                           "R-MAT scale 28, 2^32 arcs, seed 4, log2m 4"),
    "config5s": BenchConfig("config5s", 4, 42, ("harmonic",),
                            "R-MAT scale 24, 2^28 arcs (config 5 at 1/16 scale), seed 4, log2m 4"),
}


def graph_digest(g) -> str:
    """sha256 over (int64 offsets, int64 successors): independent of the id dtype."""
    h = hashlib.sha256()
    h.update(np.asarray(g.offsets, dtype=np.int64).tobytes())
    h.update(np.asarray(g.successors, dtype=np.int64).tobytes())
    return h.hexdigest()
