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


def _keys_to_device_csr(n: int, keys, dev):
    """hb_keys_to_csr on transpose keys (dst << 32 | src, self-loops ~0): sort, dedup,
    CSR -- graph.py:52-80's normalisation on the device.  Consumes `keys`."""
    import torch

    from ._lib import check, hb
    from .graph import DeviceCsrGraph
    L = hb()
    stream = torch.cuda.current_stream(dev)
    m = keys.numel()
    with torch.cuda.device(dev):
        alt = torch.empty(m, dtype=torch.int64, device=dev)
        tb = ctypes.c_uint64(0)
        mo = ctypes.c_int64(0)
        check(L.hb_keys_to_csr(n, m, keys.data_ptr(), alt.data_ptr(), None, ctypes.byref(tb),
                               ctypes.byref(mo), None, None, stream.cuda_stream), "size")
        temp = torch.empty(max(int(tb.value), 1), dtype=torch.uint8, device=dev)
        offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
        succ = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
        check(L.hb_keys_to_csr(n, m, keys.data_ptr(), alt.data_ptr(), temp.data_ptr(),
                               ctypes.byref(tb), ctypes.byref(mo), offsets.data_ptr(),
                               succ.data_ptr(), stream.cuda_stream), "hb_keys_to_csr")
        del alt, temp
        succ = succ[:mo.value].clone()
    return DeviceCsrGraph(offsets, succ)


def _device(device):
    import torch
    return torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())


def rmat_t_device(scale: int, arcs: int, seed: int, abc=RMAT_ABC, device=None):
    """rmat_t built on the GPU (hb_gen_rmat_keys + hb_keys_to_csr): the same bytes as the
    host builder (tests pin the digest), as a DeviceCsrGraph.  Peak device memory is about
    20 bytes per generated arc."""
    import torch

    from ._lib import check, hb
    dev = _device(device)
    a, b, c = abc
    thr = [int(a * 4294967296.0), int((a + b) * 4294967296.0), int((a + b + c) * 4294967296.0)]
    n = 1 << scale
    stream = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        keys = torch.empty(arcs, dtype=torch.int64, device=dev)
        check(hb().hb_gen_rmat_keys(scale, arcs, thr[0], thr[1], thr[2], seed, keys.data_ptr(),
                                    stream.cuda_stream), "hb_gen_rmat_keys")
    return _keys_to_device_csr(n, keys, dev)


_GG_ER, _GG_DISC, _GG_WEB = 1, 3, 4


def _degree_law_device(kind: int, n: int, seed: int, dev, mean: float = 0.0,
                       alpha: float = 0.0, kmin: int = 0, kmax: int = 0):
    """Per-source out-degrees drawn on the device from graphgen.c's own CDF tables, and
    their exclusive prefix sum (int64 [n+1])."""
    import torch

    from ._lib import check, hb
    G = graphlib()
    if kind == _GG_WEB:
        tab = np.empty(kmax - kmin + 1, dtype=np.float64)
        G.hbg_zipf_cdf(float(alpha), kmin, kmax, tab.ctypes.data_as(ctypes.c_void_p))
    else:
        tab = np.empty(256, dtype=np.float64)
        tab = tab[:G.hbg_poisson_cdf(float(mean), tab.ctypes.data_as(ctypes.c_void_p))].copy()
    stream = torch.cuda.current_stream(dev)
    cdf = torch.from_numpy(tab).to(dev)
    deg = torch.empty(n + 1, dtype=torch.int64, device=dev)
    check(hb().hb_gen_degrees(kind, n, seed, cdf.data_ptr(), tab.size, kmin, deg.data_ptr(),
                              stream.cuda_stream), "hb_gen_degrees")
    deg[n] = 0
    off = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(deg[:n], 0, out=off[1:])
    return off


def _arcs_device(kind, n, seed, off, dev, blo=None, bhi=None, p_local=0.0, window=1):
    import torch

    from ._lib import check, hb
    m = int(off[-1].item())
    stream = torch.cuda.current_stream(dev)
    keys = torch.empty(max(m, 1), dtype=torch.int64, device=dev)[:m]
    check(hb().hb_gen_arc_keys(kind, n, seed, off.data_ptr(),
                               blo.data_ptr() if blo is not None else None,
                               bhi.data_ptr() if bhi is not None else None, float(p_local),
                               int(window), keys.data_ptr(), stream.cuda_stream),
          "hb_gen_arc_keys")
    return _keys_to_device_csr(n, keys, dev)


def erdos_renyi_t_device(n: int, mean_degree: float, seed: int, device=None):
    """erdos_renyi_t built on the GPU (same bytes as the host builder)."""
    import torch
    dev = _device(device)
    with torch.cuda.device(dev):
        off = _degree_law_device(_GG_ER, n, seed, dev, mean=mean_degree)
        return _arcs_device(_GG_ER, n, seed, off, dev)


def disconnected_t_device(n: int, giant: int, geo_p: float, mean_degree: float, seed: int,
                          device=None):
    """disconnected_t built on the GPU (same bytes as the host builder): block sizes drawn
    for every possible block in parallel, prefix-summed into block bounds."""
    import torch

    from ._lib import check, hb
    dev = _device(device)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        nb = max(n - giant, 0)
        size = torch.empty(max(nb, 1), dtype=torch.int64, device=dev)
        start = torch.empty(max(nb, 1), dtype=torch.int64, device=dev)
        blo = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        bhi = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        tb = ctypes.c_uint64(0)
        check(hb().hb_gen_blocks(n, giant, float(geo_p), seed, size.data_ptr(), start.data_ptr(),
                                 blo.data_ptr(), bhi.data_ptr(), None, ctypes.byref(tb),
                                 stream.cuda_stream), "hb_gen_blocks(size)")
        temp = torch.empty(max(int(tb.value), 1), dtype=torch.uint8, device=dev)
        check(hb().hb_gen_blocks(n, giant, float(geo_p), seed, size.data_ptr(), start.data_ptr(),
                                 blo.data_ptr(), bhi.data_ptr(), temp.data_ptr(),
                                 ctypes.byref(tb), stream.cuda_stream), "hb_gen_blocks")
        del size, start, temp
        off = _degree_law_device(_GG_DISC, n, seed, dev, mean=mean_degree)
        return _arcs_device(_GG_DISC, n, seed, off, dev, blo, bhi)


def weblike_t_device(n: int, seed: int, alpha: float = 2.1, kmin: int = 3, kmax: int = 10_000,
                     p_local: float = 0.8, window: int = 1024, device=None):
    """weblike_t built on the GPU (same bytes as the host builder)."""
    import torch
    dev = _device(device)
    with torch.cuda.device(dev):
        off = _degree_law_device(_GG_WEB, n, seed, dev, alpha=alpha, kmin=kmin, kmax=kmax)
        return _arcs_device(_GG_WEB, n, seed, off, dev, p_local=p_local, window=window)


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
        """The graph built on the GPU (every config has a device builder producing the
        host builder's bytes), as a DeviceCsrGraph."""
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
    "config1": lambda dev=None: erdos_renyi_t_device(10_000, 8.0, seed=0, device=dev),
    "config3": lambda dev=None: disconnected_t_device(1 << 22, 1 << 21, 0.1, 6.0, seed=2,
                                                      device=dev),
    "config4": lambda dev=None: weblike_t_device(1 << 24, seed=3, device=dev),
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
