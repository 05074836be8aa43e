"""Randomised parity sweep: seeded random graphs of many shapes -- empty rows, isolated
nodes, self-loops and duplicate arcs, power-law hubs that take the heavy path, long chains
that converge late -- at every supported b, register widths 5-8, every schedule order,
with and without the per-source skip, single device and simulated ranks with both
exchanges; every run is compared with the CPU oracle after EVERY iteration (registers,
estimates, changed count) and in its centralities, bit for bit."""

import hashlib

import numpy as np
import pytest

import oracle as orc

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_1308_2144_b200")
from paper_1308_2144_b200.distributed import run_simulated  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def random_graph(seed):
    """G^T CSR of a random multigraph (transpose of the arc list the reference would be
    given: self-loops and duplicates kept, graph.py:145-155)."""
    rng = np.random.default_rng(seed)
    kind = seed % 4
    n = int(rng.integers(1, 6000))
    if kind == 0:                                   # uniform, some empty rows
        m = int(rng.integers(0, 8 * n))
        src, dst = rng.integers(0, n, m), rng.integers(0, n, m)
    elif kind == 1:                                 # power-law in-degree: hubs
        m = int(rng.integers(n, 12 * n))
        src = rng.integers(0, n, m)
        dst = np.minimum((rng.pareto(1.2, m) * 3).astype(np.int64), n - 1)
    elif kind == 2:                                 # chains + a few shortcuts: late convergence
        n = min(n, 400)                             # (one iteration per chain link)
        s = np.arange(n - 1)
        extra = int(rng.integers(0, n // 10 + 1))
        src = np.concatenate([s, rng.integers(0, n, extra)])
        dst = np.concatenate([s + 1, rng.integers(0, n, extra)])
    else:                                           # islands with self-loops and duplicates
        block = int(rng.integers(2, 50))
        m = int(rng.integers(n, 5 * n))
        src = rng.integers(0, n, m)
        dst = np.clip(src + rng.integers(-block, block + 1, m), 0, n - 1)
        dup = rng.integers(0, max(m, 1), m // 10)
        src, dst = np.concatenate([src, src[dup]]), np.concatenate([dst, dst[dup]])
    g = hb.CsrGraph.from_edges(src, dst, n=n)
    gt = hb.transpose(g)
    return np.asarray(gt.offsets, np.int64), np.asarray(gt.successors, np.int64)


def run_gpu(off, suc, b, seed, width, schedule, skip):
    g = hb.CsrGraph(off, suc)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=b, register_width=width, seed=seed),
                             schedule=schedule, skip_stable_nodes=skip)
    acc = hb.CentralityAccumulator(g.n)
    st = hb.initialize(g, cfg)
    regs, ests, nchs = [sha(st.register_matrix())], [sha(st.est)], []
    while g.n:
        nch = hb.iterate(g, st, [acc])
        regs.append(sha(st.register_matrix()))
        ests.append(sha(st.est))
        nchs.append(nch)
        if nch == 0:
            break
    acc.on_converged(st.est)
    return st, acc, regs, ests, nchs


@pytest.mark.parametrize("seed", range(64))
def test_random_graph_vs_oracle(seed):
    off, suc = random_graph(seed)
    rng = np.random.default_rng(1000 + seed)
    b = int(rng.integers(4, 13))
    width = int(rng.choice([5, 5, 6, 8]))
    schedule = ["auto", "identity", "degree", "window"][seed % 4]
    skip = bool(seed % 5)
    hseed = int(rng.integers(0, 2**63))
    want = orc.run_oracle(off, suc, b, hseed, width=width, workers=4, skip=skip)
    st, acc, regs, ests, nchs = run_gpu(off, suc, b, hseed, width, schedule, skip)
    assert st.t == want.t
    assert nchs == want.nch
    assert regs == want.reg_digests
    assert ests == want.est_digests
    for fin, arr in ((hb.finalize_harmonic, want.harmonic), (hb.finalize_closeness,
                     want.closeness), (hb.finalize_lin, want.lin)):
        assert np.array_equal(fin(acc).view(np.uint64), arr.view(np.uint64)), fin.__name__


@pytest.mark.parametrize("seed", range(32))
def test_random_graph_simulated_ranks(seed):
    off, suc = random_graph(100 + seed)
    rng = np.random.default_rng(2000 + seed)
    b = int(rng.integers(4, 9))
    world = int(rng.integers(2, 6))
    exchange = ["push", "allgather"][seed % 2]
    schedule = ["identity", "degree", "window"][seed % 3]
    hseed = int(rng.integers(0, 2**63))
    want = orc.run_oracle(off, suc, b, hseed, workers=4)
    g = hb.CsrGraph(off, suc)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=b, seed=hseed), schedule=schedule)
    acc = hb.CentralityAccumulator(g.n)
    res = run_simulated(g, cfg, world, [acc], exchange=exchange)
    assert res.t == want.t
    for r in res.registers:
        assert sha(r) == want.reg_digests[-1]
    assert np.array_equal(hb.finalize_harmonic(acc).view(np.uint64),
                          want.harmonic.view(np.uint64))
