"""The per-arc dense rule (engine.DENSE_ARC_FRAC): a step merges every source without the
per-source test when the sampled share of arcs whose source changed is high.  Merging an
unchanged source is a no-op, so any rule gives identical results; the sampler must track
the exact share."""

import hashlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_1308_2144_b200")
from paper_1308_2144_b200 import _lib  # noqa: E402
from paper_1308_2144_b200 import engine as eng  # noqa: E402
from paper_1308_2144_b200 import generators as gen  # noqa: E402


@pytest.fixture(scope="module")
def rmat():
    return gen.rmat_t(14, 16 << 14, seed=7)


def _run(g, b, monkeypatch, frac, min_arcs=0):
    monkeypatch.setattr(eng, "DENSE_ARC_FRAC", frac)
    monkeypatch.setattr(eng, "FLAG_MIN_ARCS", min_arcs)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=b, seed=42))
    acc = hb.CentralityAccumulator(g.n)
    st = hb.initialize(g, cfg)
    digests, flags = [], []
    while True:
        nch = hb.iterate(g, st, [acc])
        digests.append(hashlib.sha256(st.register_matrix().tobytes()).hexdigest())
        flags.append(st._dev.last_flagged)
        if nch == 0:
            break
    acc.on_converged(st.est)
    return st.t, digests, hb.finalize_harmonic(acc), hb.finalize_lin(acc), flags


@pytest.mark.parametrize("b", [4, 7])
def test_rule_does_not_change_results(rmat, b, monkeypatch):
    base = _run(rmat, b, monkeypatch, 1.0)          # per-arc rule off
    for frac in (0.0, 0.5):                        # 0.0: every step dense
        got = _run(rmat, b, monkeypatch, frac)
        assert got[0] == base[0] and got[1] == base[1]
        for x, y in ((got[2], base[2]), (got[3], base[3])):
            assert np.array_equal(x.view(np.uint64), y.view(np.uint64))
        assert all(f is not None for f in got[4])


def test_sampled_share_tracks_exact(rmat):
    dv = torch.device("cuda", 0)
    off = torch.from_numpy(np.asarray(rmat.offsets, np.int64)).to(dv)
    suc = torch.from_numpy(np.asarray(rmat.successors, np.int32)).to(dv)
    n, m = rmat.n, int(suc.numel())
    rng = np.random.default_rng(3)
    for p_flag in (0.02, 0.3, 0.9):
        flags = rng.random(n) < p_flag
        words = np.zeros((n + 31) // 32, np.uint32)
        idx = np.flatnonzero(flags)
        np.bitwise_or.at(words, idx >> 5, (1 << (idx & 31)).astype(np.uint32))
        bits = torch.from_numpy(words.view(np.int32)).to(dv)
        out = torch.zeros(1, dtype=torch.int64, device=dv)
        samples = 1 << 16
        _lib.check(_lib.hb().hb_sample_flagged_arcs(
            m, suc.data_ptr(), bits.data_ptr(), samples, 5, out.data_ptr(),
            torch.cuda.current_stream().cuda_stream), "hb_sample_flagged_arcs")
        est = int(out.item()) / samples
        exact = flags[np.asarray(rmat.successors)].mean()
        assert abs(est - exact) < 0.02, (p_flag, est, exact)
    del off
