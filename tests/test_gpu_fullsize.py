"""Parity at BASELINE.json's full sizes (configs 1-5, and config 5 at 1/16 scale) against
the CPU oracle run on the same generated graph on the GPU box's host cores.

Checked bit for bit: the changed count of every iteration, the sha256 of the estimate
array after every iteration, the iteration count, the final register matrix, and the
final harmonic / closeness / Lin arrays.  Size-independent properties are checked too:
registers are monotone between iterations and never exceed the saturation value.
"""

import hashlib
import os

import numpy as np
import pytest

import oracle as orc

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_1308_2144_b200")
from paper_1308_2144_b200 import generators as gen  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def oracle_run(g, b, seed):
    """run_oracle with per-iteration estimate digests only (registers compared at the end)."""
    off = np.asarray(g.offsets, np.int64)
    suc = np.asarray(g.successors, np.int64)
    n = g.n
    threads = os.cpu_count() or 1
    cur, est = orc.seed_registers(n, b, 5, seed)
    chg = np.ones(n, np.uint8)
    sd, sr = np.zeros(n), np.zeros(n)
    nch_list, est_d = [], [sha(est)]
    import ctypes
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    L = orc.lib()
    nxt = np.zeros_like(cur)
    now = np.zeros(n, np.uint8)
    new = np.zeros(n)
    t = 0
    while True:
        nch = L.orc_iterate_range_mt(0, n, P(off), P(suc), P(cur), P(nxt), P(chg), P(now),
                                     P(est), P(new), b, 1, threads)
        t += 1
        L.orc_accumulate(n, t, P(est), P(new), P(sd), P(sr))
        cur, nxt = nxt, cur
        est, new = new, est
        chg, now = now, chg
        nch_list.append(int(nch))
        est_d.append(sha(est))
        if nch == 0:
            break
    clo, har, lin = np.zeros(n), np.zeros(n), np.zeros(n)
    L.orc_finalize(n, P(sd), P(sr), P(est), P(clo), P(har), P(lin))
    return dict(t=t, nch=nch_list, est_d=est_d, regs=cur, clo=clo, har=har, lin=lin)


@pytest.mark.parametrize("name", ["config1", "config2", "config3", "config4", "config5s",
                                  "config5"])
def test_full_size_config_vs_oracle(name):
    cfgd = gen.CONFIGS[name]
    if name == "config5":
        # 2^32 arcs: built on the device (byte-identical to the host builder) and copied
        # out; the oracle then needs ~50 GB of host memory and about a minute
        import torch
        g = cfgd.build_device(torch.device("cuda", 0)).to_host()
        torch.cuda.empty_cache()
    else:
        g = cfgd.build()
    ref = oracle_run(g, cfgd.log2m, cfgd.hash_seed)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=cfgd.log2m, seed=cfgd.hash_seed))
    acc = hb.CentralityAccumulator(g.n)
    st = hb.initialize(g, cfg)
    est_d, nchs = [sha(st.est)], []
    prev = st.register_matrix()
    sat = cfg.params.saturation
    while True:
        nch = hb.iterate(g, st, [acc])
        nchs.append(nch)
        est_d.append(sha(st.est))
        if st.t in (1, 2, ref["t"] // 2):         # size-independent properties, sampled
            regs = st.register_matrix()
            assert (regs >= prev).all() and int(regs.max()) <= sat
            prev = regs
        if nch == 0:
            break
    acc.on_converged(st.est)
    assert st.t == ref["t"]
    assert nchs == ref["nch"]
    assert est_d == ref["est_d"]
    assert np.array_equal(st.register_matrix(), ref["regs"])
    for got, want in ((hb.finalize_harmonic(acc), ref["har"]),
                      (hb.finalize_closeness(acc), ref["clo"]),
                      (hb.finalize_lin(acc), ref["lin"])):
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_config5_full_scale_sampled():
    """Config 5 itself (R-MAT scale 28, 2^32 arcs, p = 16) is too large for the CPU oracle
    here, so the first iterations are checked on 20 000 random nodes: each new row must
    be the byte-wise max of the node's previous row and its in-neighbours' previous rows
    (_kernels.py:67-114; merging an unchanged source is a no-op), and its estimate the
    oracle's estimate of that row (_kernels.py:15-34), bit for bit."""
    import torch
    dev = torch.device("cuda", 0)
    g = gen.CONFIGS["config5"].build_device(dev)
    n = g.n
    st = hb.initialize(g, hb.HyperBallConfig(params=hb.CounterParams(b=4, seed=42), device=0))
    rng = np.random.default_rng(5)
    vs = np.sort(rng.choice(n, 20_000, replace=False))
    vt = torch.from_numpy(vs).to(dev)
    beg, end = g.offsets[vt], g.offsets[vt + 1]
    lens = end - beg
    starts = torch.cumsum(lens, 0) - lens
    total = int(lens.sum().item())
    pos = torch.repeat_interleave(beg - starts, lens) + torch.arange(total, device=dev)
    ids = g.successors[pos].long().cpu().numpy()
    seg = np.repeat(np.arange(vs.size), lens.cpu().numpy())
    for _ in range(3):
        before = st.register_matrix()
        hb.iterate(g, st, [])
        after = st.register_matrix()
        want = before[vs].copy()
        np.maximum.at(want, seg, before[ids])
        assert np.array_equal(after[vs], want)
        assert np.array_equal(st.est[vs].view(np.uint64),
                              orc.estimate_rows(want, 4).view(np.uint64))
        assert int(after.max()) <= 31
        del before, after
