"""Fixtures for the graph-build path produced by the REFERENCE:
``CsrGraph.from_edges`` (graph.py:52-80) and ``transpose`` (graph.py:145-155) on forward
graphs with duplicate arcs, self-loops, isolated nodes and empty rows.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_transpose_golden.py

Writes tests/golden/transpose.npz: for every case the forward CSR (offsets,
successors; some built directly as multigraphs, bypassing from_edges' dedup) and the
reference's transpose; for the arc-list cases also the raw arc arrays and
from_edges(src, dst, n) itself.  The CPU tests check graph.transpose against it, the GPU
tests hb_transpose_csr and the device graph builders.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
import hyperball as ref  # noqa: E402


def main():
    out = {}
    rng = np.random.default_rng(2024)
    cases = []
    for name, n, m in (("tiny", 5, 9), ("r200", 200, 900), ("r3000", 3000, 20000),
                       ("sparse5000", 5000, 2500), ("dense64", 64, 3000)):
        src = rng.integers(0, n, m)
        dst = rng.integers(0, n, m)
        out[f"{name}/arcs_src"], out[f"{name}/arcs_dst"] = src, dst
        g = ref.CsrGraph.from_edges(src, dst, n=n)          # sorted, deduplicated
        out[f"{name}/from_edges_offsets"] = g.offsets
        out[f"{name}/from_edges_successors"] = g.successors
        keep = src != dst                                   # the synthetic builders' rule
        gt = ref.transpose(ref.CsrGraph.from_edges(src[keep], dst[keep], n=n))
        out[f"{name}/noloop_t_offsets"] = gt.offsets
        out[f"{name}/noloop_t_successors"] = gt.successors
        cases.append((name, g))
    # multigraph: duplicate arcs and self-loops kept, rows unsorted (raw CsrGraph)
    n = 400
    deg = rng.integers(0, 9, n)
    deg[::7] = 0
    off = np.zeros(n + 1, np.int64)
    np.cumsum(deg, out=off[1:])
    suc = rng.integers(0, n, int(off[-1]))
    suc[::5] = np.repeat(np.arange(n), deg)[::5]           # self-loops
    suc[1::11] = suc[0:-1:11][:suc[1::11].size]            # duplicates
    cases.append(("multi400", ref.CsrGraph(off, suc)))
    cases.append(("empty7", ref.CsrGraph(np.zeros(8, np.int64), np.zeros(0, np.int64))))
    for name, g in cases:
        t = ref.transpose(g)
        out[f"{name}/offsets"], out[f"{name}/successors"] = g.offsets, g.successors
        out[f"{name}/t_offsets"], out[f"{name}/t_successors"] = t.offsets, t.successors
        print(name, g.n, g.m)
    out["names"] = np.array([c[0] for c in cases])
    np.savez_compressed(os.path.join(HERE, "transpose.npz"), **out)


if __name__ == "__main__":
    main()
