"""Streamed upload (schedule.py STREAM_SLICES): the successor ids arrive in row slices and
iteration 1 runs slice by slice (window relabel per slice for the window order).  Every
result must equal the unstreamed run bit for bit, and the oracle's."""

import hashlib
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_1308_2144_b200")
from paper_1308_2144_b200 import generators as gen  # noqa: E402
from paper_1308_2144_b200 import schedule as sched_mod  # noqa: E402

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle"))


@pytest.fixture(scope="module")
def weblike():
    g = gen.weblike_t(1 << 15, seed=5)
    assert np.asarray(g.successors).dtype == np.int32
    return g


def _run(g, b, schedule, slices, monkeypatch, skip=True):
    monkeypatch.setattr(sched_mod, "STREAM_SLICES", slices)
    monkeypatch.setattr(sched_mod, "STREAM_MIN_ARCS", 0)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=b, seed=42), schedule=schedule,
                             skip_stable_nodes=skip)
    acc = hb.CentralityAccumulator(g.n)
    st = hb.initialize(g, cfg)
    pending = len(st._dev.sched.pending)
    digests = []
    while True:
        nch = hb.iterate(g, st, [acc])
        digests.append(hashlib.sha256(st.register_matrix().tobytes()).hexdigest())
        if nch == 0:
            break
    acc.on_converged(st.est)
    out = dict(t=st.t, digests=digests, est=st.est,
               h=hb.finalize_harmonic(acc), c=hb.finalize_closeness(acc),
               lin=hb.finalize_lin(acc), merged=st._dev.merged_total)
    return out, pending, st


def _same(a, b):
    assert a["t"] == b["t"]
    assert a["digests"] == b["digests"]
    assert a["merged"] == b["merged"]
    for k in ("est", "h", "c", "lin"):
        assert np.array_equal(a[k].view(np.uint64), b[k].view(np.uint64)), k


@pytest.mark.parametrize("schedule", ["window", "identity"])
@pytest.mark.parametrize("slices", [3, 8])
def test_streamed_equals_unstreamed(weblike, schedule, slices, monkeypatch):
    ref, pend0, _ = _run(weblike, 8, schedule, 1, monkeypatch)
    got, pend, st = _run(weblike, 8, schedule, slices, monkeypatch)
    assert pend0 == 0 and pend > 1                 # the streamed path really ran
    assert not st._dev.sched.pending
    _same(got, ref)


def test_streamed_matches_oracle(weblike, monkeypatch):
    import oracle as orc
    got, pend, _ = _run(weblike, 6, "window", 5, monkeypatch)
    assert pend > 1
    ref = orc.run_oracle(np.asarray(weblike.offsets, np.int64),
                         np.asarray(weblike.successors, np.int64), 6, 42, workers=4)
    assert got["t"] == ref.t
    assert got["digests"] == ref.reg_digests[1:]
    for k, want in (("h", ref.harmonic), ("c", ref.closeness), ("lin", ref.lin)):
        assert np.array_equal(got[k].view(np.uint64), want.view(np.uint64)), k


@pytest.mark.parametrize("slices", [2, 6])
def test_degree_order_relabels_by_slice(weblike, slices, monkeypatch):
    """Degree order: every slice is relabelled (scatter form) as it lands; iteration 1
    starts after the last one."""
    ref, _, _ = _run(weblike, 7, "degree", 1, monkeypatch)
    got, pend, _ = _run(weblike, 7, "degree", slices, monkeypatch)
    assert pend == 0
    _same(got, ref)


def test_degree_order_rmat_streamed(monkeypatch):
    """Skewed in-degree (heavy items) with the per-slice degree relabel."""
    g = gen.rmat_t(13, 16 << 13, seed=3)
    ref, _, _ = _run(g, 4, "degree", 1, monkeypatch)
    got, _, _ = _run(g, 4, "degree", 5, monkeypatch)
    _same(got, ref)


def test_reader_before_first_step_finishes_slices(weblike, monkeypatch):
    """Anything that reads the CSR before iteration 1 (through Schedule.succ) sees every
    slice uploaded and relabelled; the run then proceeds unsliced."""
    monkeypatch.setattr(sched_mod, "STREAM_SLICES", 4)
    monkeypatch.setattr(sched_mod, "STREAM_MIN_ARCS", 0)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=8, seed=42), schedule="window")
    st = hb.initialize(weblike, cfg)
    s = st._dev.sched
    assert len(s.pending) > 1
    _ = s.succ                                     # property: finishes every slice
    assert not s.pending and s.relabel is None
    hb.resume(weblike, st)
    monkeypatch.setattr(sched_mod, "STREAM_SLICES", 1)
    ref = hb.run(weblike, cfg)
    assert st.t == ref.t
    assert np.array_equal(st.register_matrix(), ref.register_matrix())


def test_skip_off_streamed(weblike, monkeypatch):
    ref, _, _ = _run(weblike, 5, "window", 1, monkeypatch, skip=False)
    got, pend, _ = _run(weblike, 5, "window", 4, monkeypatch, skip=False)
    assert pend > 1
    _same(got, ref)


def test_int64_ids_streamed(weblike, monkeypatch):
    """The reference's CsrGraph carries int64 ids: streamed too, narrowed on the device."""
    g64 = hb.CsrGraph(np.asarray(weblike.offsets, np.int64),
                      np.asarray(weblike.successors, np.int64))
    ref, _, _ = _run(weblike, 8, "window", 1, monkeypatch)
    got, pend, _ = _run(g64, 8, "window", 5, monkeypatch)
    assert pend > 1
    _same(got, ref)


@pytest.mark.parametrize("seed", range(6))
def test_streamed_random_small_graphs(seed, monkeypatch):
    """Corner cases of the slicing: tiny and ragged graphs (isolated nodes, empty slices,
    n not a multiple of the window), every order and several widths."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(50, 3000))
    m = int(rng.integers(0, 8 * n))
    src, dst = rng.integers(0, n, m), rng.integers(0, n, m)
    if seed % 2:                                 # hub-heavy variant: heavy items
        dst[: m // 3] = rng.integers(0, 4, m // 3)
    g = gen.from_arcs_t(n, src, dst)
    b = int(rng.choice([4, 6, 8]))
    for schedule in ("window", "identity", "degree"):
        ref, _, _ = _run(g, b, schedule, 1, monkeypatch)
        got, _, _ = _run(g, b, schedule, int(rng.integers(2, 17)), monkeypatch)
        _same(got, ref)


@pytest.mark.parametrize("dtype", ["int32", "int64"])
@pytest.mark.parametrize("pinned", [True, False])
def test_staged_and_pinned_uploads(weblike, dtype, pinned, monkeypatch):
    """The two upload routes of the streamed path: pinned int32 ids are copied as they
    are; pageable or int64 ids (the reference's CsrGraph) go through the pinned staging
    ring (hbg_stage_ids narrows on every core); pageable int64 offsets through
    hbg_stage_bytes.  Both equal the unstreamed run bit for bit."""
    import torch
    ref, _, _ = _run(weblike, 8, "window", 1, monkeypatch)
    off = np.asarray(weblike.offsets, np.int64)
    suc = np.asarray(weblike.successors).astype(dtype)
    if pinned:
        po = torch.empty(off.shape[0], dtype=torch.int64, pin_memory=True)
        po.numpy()[:] = off
        ps = torch.empty(suc.shape[0], dtype=getattr(torch, dtype), pin_memory=True)
        ps.numpy()[:] = suc
        off, suc = po.numpy(), ps.numpy()
    got, pend, _ = _run(hb.CsrGraph(off, suc), 8, "window", 5, monkeypatch)
    assert pend > 1
    _same(ref, got)
    # offsets above the staging threshold also take the staged route
    big = np.zeros((1 << 20) + 1, np.int64)
    t = sched_mod._upload_offsets(big, torch.device("cuda", 0),
                                  torch.cuda.current_stream())
    torch.cuda.synchronize()
    assert t.shape[0] == big.shape[0] and int(t.abs().sum().item()) == 0


def test_release_staging_buffers(weblike, monkeypatch):
    """The pinned staging buffers of a pageable upload are kept for the next run and freed
    on request (after their copies completed); a run afterwards allocates them again."""
    ref, _, _ = _run(weblike, 8, "window", 1, monkeypatch)
    got, _, _ = _run(hb.CsrGraph(np.asarray(weblike.offsets, np.int64),
                                 np.asarray(weblike.successors, np.int64)), 8, "window", 4,
                     monkeypatch)
    assert sched_mod._STAGING
    hb.release_staging_buffers()
    assert not sched_mod._STAGING
    again, _, _ = _run(hb.CsrGraph(np.asarray(weblike.offsets, np.int64),
                                   np.asarray(weblike.successors, np.int64)), 8, "window", 4,
                       monkeypatch)
    _same(ref, got)
    _same(ref, again)
