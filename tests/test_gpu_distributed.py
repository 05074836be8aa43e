"""Multi-rank path on one GPU: every rank simulated in one process, phase by phase
(local union step, refresh of remote rows, hb_gather_changed, exchange, hb_scatter_rows).
Registers, estimates, iteration count and centralities must be bit-identical to the
reference (golden) for every world size -- the worker-count invariance of
test_engine.py:231-239 lifted to GPUs."""

import hashlib

import numpy as np
import pytest

from conftest import golden, golden_cases, golden_graph

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_1308_2144_b200")
from paper_1308_2144_b200 import generators as gen  # noqa: E402
from paper_1308_2144_b200.distributed import run_simulated  # noqa: E402

CASES = {c["key"]: c for c in golden_cases()}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("packed", [True, False])
@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("schedule", ["identity", "degree", "window"])
@pytest.mark.parametrize("key", ["random300_b6_s42_w5", "disc14_b4_s42_w5", "rmat12_b7_s42_w5",
                                 "config1_b6_s42_w5", "sparse2000_b4_s42_w5",
                                 "web14_b8_s42_w5"])
def test_simulated_ranks_match_reference(key, world, schedule, packed):
    case = CASES[key]
    off, suc = golden_graph(case)
    g = hb.CsrGraph(off, suc)
    acc = hb.CentralityAccumulator(g.n)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=case["b"], seed=int(case["seed"])),
                             schedule=schedule)
    res = run_simulated(g, cfg, world, [acc], packed=packed)
    assert res.t == case["t"]
    for regs in res.registers:        # every replica holds the final registers
        assert sha(regs) == case["reg_digests"][-1]
    assert sha(res.est) == case["est_digests"][-1]
    _, arrays = golden()
    for name, got in (("harmonic", hb.finalize_harmonic(acc)), ("lin", hb.finalize_lin(acc)),
                      ("closeness", hb.finalize_closeness(acc))):
        assert np.array_equal(got.view(np.uint64), arrays[f"{key}/{name}"].view(np.uint64))


def test_simulated_heavy_rmat_matches_single_gpu():
    g = gen.rmat_t(15, 16 << 15, seed=31)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=5, seed=3))
    a1 = hb.CentralityAccumulator(g.n)
    st = hb.run(g, cfg, [a1])
    a4 = hb.CentralityAccumulator(g.n)
    res = run_simulated(g, cfg, 4, [a4])
    assert res.t == st.t
    assert sha(res.registers[0]) == sha(st.register_matrix())
    assert np.array_equal(a1.sum_recip.view(np.uint64), a4.sum_recip.view(np.uint64))


@pytest.mark.parametrize("packed", [True, False])
@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("schedule", ["identity", "degree"])
@pytest.mark.parametrize("key", ["random300_b6_s42_w5", "disc14_b4_s42_w5", "rmat12_b7_s42_w5",
                                 "config1_b6_s42_w5", "web14_b8_s42_w5"])
def test_fused_push_matches_reference(key, world, schedule, packed):
    """The fused push (hb_union_step storing rows and change bits into every peer's
    replica -- or 5-bit packed into the peers' inboxes, unpacked after the step) on
    simulated ranks: bit-identical to the reference."""
    case = CASES[key]
    off, suc = golden_graph(case)
    g = hb.CsrGraph(off, suc)
    acc = hb.CentralityAccumulator(g.n)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=case["b"], seed=int(case["seed"])),
                             schedule=schedule)
    res = run_simulated(g, cfg, world, [acc], exchange="push", packed=packed)
    assert res.t == case["t"]
    for regs in res.registers:
        assert sha(regs) == case["reg_digests"][-1]
    assert sha(res.est) == case["est_digests"][-1]
    _, arrays = golden()
    assert np.array_equal(hb.finalize_lin(acc).view(np.uint64),
                          arrays[f"{key}/lin"].view(np.uint64))


_ONE_RANK = r"""
import hashlib, json, sys
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, sys.argv[1])
import paper_1308_2144_b200 as hb
from paper_1308_2144_b200.distributed import CudaRankState, SymmetricBuffers, iterate_push
dist.init_process_group("nccl", init_method="tcp://127.0.0.1:" + sys.argv[2], rank=0,
                        world_size=1, device_id=torch.device("cuda", 0))
d = np.load(sys.argv[3])
g = hb.CsrGraph(d["off"], d["suc"])
cfg = hb.HyperBallConfig(params=hb.CounterParams(b=int(sys.argv[4]), seed=int(sys.argv[5])),
                         schedule=sys.argv[6])
st = CudaRankState(g, cfg, 1, 0)
symm = SymmetricBuffers(st)
t = 0
while True:
    t += 1
    nch = iterate_push(st, symm, t, t == 1)
    if nch == 0:
        break
regs = st.dev.to_host(st.dev.cur)
est = st.dev.to_host(st.dev.est)
print(json.dumps({"t": t, "regs": hashlib.sha256(regs.tobytes()).hexdigest(),
                  "est": hashlib.sha256(np.ascontiguousarray(est).tobytes()).hexdigest()}))
dist.destroy_process_group()
"""


@pytest.mark.parametrize("schedule", ["identity", "degree"])
def test_symmetric_buffers_one_rank(tmp_path, schedule):
    """The real fused-push plumbing (symmetric-memory double buffer, NCCL all-reduce as
    the barrier) on a one-rank NCCL group in a subprocess: the seeded buffers are carried
    into symmetric memory (incl. rows iteration 1 skips) and the run matches the golden."""
    import json
    import os
    import socket
    import subprocess
    import sys
    case = CASES["rmat12_b7_s42_w5"]
    off, suc = golden_graph(case)
    path = tmp_path / "g.npz"
    np.savez(path, off=off, suc=suc)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", _ONE_RANK, repo, str(port), str(path), "7", "42",
                          schedule], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["t"] == case["t"]
    assert res["regs"] == case["reg_digests"][-1]
    assert res["est"] == case["est_digests"][-1]


@pytest.mark.parametrize("world", [1, 3, 8])
@pytest.mark.parametrize("key", ["star6_b7_s42_w5", "path8_b4_s42_w5", "config1_b4_b4_s42_w5",
                                 "dag300_b4_s42_w6_nw3", "rmat12_b7_s42_w5"])
def test_always_dense_steps(key, world, monkeypatch):
    """Dense steps (every source merged, no per-source change test) give the reference's
    bits in every iteration, single-GPU and on simulated ranks with the fused push --
    merging an unchanged source is a no-op only if every replica row is current, which
    is what this checks (the engine goes dense when >= 95% of the counters changed)."""
    from paper_1308_2144_b200 import distributed as D
    from paper_1308_2144_b200 import engine as E
    monkeypatch.setattr(E, "DENSE_FRAC", 0.0)
    monkeypatch.setattr(D, "DENSE_FRAC", 0.0)
    case = CASES[key]
    off, suc = golden_graph(case)
    _, arrays = golden()
    w = arrays[f"{key}/weights"] if case.get("weights_seed") is not None else None
    g = hb.CsrGraph(off, suc)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=case["b"], seed=int(case["seed"]),
                                                     register_width=case["width"]),
                             schedule="degree", weights=w)
    if world == 1:
        st = hb.run(g, cfg)
        assert st.t == case["t"] and sha(st.register_matrix()) == case["reg_digests"][-1]
        return
    res = run_simulated(g, cfg, world, [], exchange="push")
    assert res.t == case["t"]
    for regs in res.registers:
        assert sha(regs) == case["reg_digests"][-1]


DISC_KEYS = [c["key"] for c in golden_cases() if c.get("discounts")]


@pytest.mark.parametrize("exchange", ["allgather", "push"])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("key", DISC_KEYS)
def test_simulated_ranks_fused_discounts(key, world, exchange):
    """Discounted gains (centrality.py:26-101,149-150) folded in every rank's union
    epilogue and gathered back: bit-identical to the reference's host accumulation."""
    case = CASES[key]
    off, suc = golden_graph(case)
    g = hb.CsrGraph(off, suc)
    specs = [hb.DiscountSpec.preset(name) if tab is None
             else hb.DiscountSpec.from_table(tab[0], tab[1], name="table")
             for name, tab in case["discounts"]]
    acc = hb.CentralityAccumulator(g.n, specs)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=case["b"], seed=int(case["seed"])))
    res = run_simulated(g, cfg, world, [acc], exchange=exchange)
    assert res.t == case["t"]
    _, arrays = golden()
    for spec in specs:
        got = hb.finalize_discounted(acc, spec.name)
        want = arrays[f"{key}/disc_{spec.name}"]
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), spec.name
    assert np.array_equal(hb.finalize_harmonic(acc).view(np.uint64),
                          arrays[f"{key}/harmonic"].view(np.uint64))


@pytest.mark.parametrize("slices", [1, 5])
@pytest.mark.parametrize("on_device", [False, True])
@pytest.mark.parametrize("schedule", ["identity", "degree", "window"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_rank_local_csr(world, schedule, on_device, slices, monkeypatch):
    """Every rank holds only the successor ids of the rows it owns (~m/W, uploaded -- in
    `slices` streamed slices from the host -- or gathered alone), ids in the internal order;
    the union over ranks is the graph, and the simulated-rank run stays bit-identical to
    the reference."""
    import torch
    from paper_1308_2144_b200 import schedule as sched_mod
    if on_device and slices > 1:
        pytest.skip("streamed slices are a host-upload feature")
    monkeypatch.setattr(sched_mod, "STREAM_SLICES", slices)
    monkeypatch.setattr(sched_mod, "STREAM_MIN_ARCS", 0)
    from paper_1308_2144_b200.distributed import CudaRankState
    from paper_1308_2144_b200.schedule import partition_bounds
    case = CASES["rmat12_b7_s42_w5"]
    off, suc = golden_graph(case)
    g = (hb.DeviceCsrGraph(torch.from_numpy(off).cuda(),
                           torch.from_numpy(suc.astype(np.int32)).cuda())
         if on_device else hb.CsrGraph(off, suc))
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=case["b"], seed=int(case["seed"])),
                             schedule=schedule)
    states = [CudaRankState(g, cfg, world, r) for r in range(world)]
    bounds = partition_bounds(g.n, world)
    deg = np.diff(off)
    total = 0
    for r, st in enumerate(states):
        s = st.dev.sched
        pad = bounds[r] - s.row_base
        assert s.local and 0 <= pad < 64 and s.lo == bounds[r]
        assert s.offsets.numel() == bounds[r + 1] - s.row_base + 1
        perm = (s.perm.cpu().numpy() if s.perm is not None
                else np.arange(g.n, dtype=np.int32))
        rank = np.empty(g.n, np.int64)
        rank[perm] = np.arange(g.n)
        mine = perm[bounds[r]:bounds[r + 1]]
        assert s.m == int(deg[mine].sum())                  # only this rank's arcs
        lo_off = s.offsets.cpu().numpy()[pad:]
        ids = s.succ.cpu().numpy()
        for i in range(0, mine.size, max(1, mine.size // 50)):
            row = np.sort(ids[lo_off[i]:lo_off[i + 1]])
            want = np.sort(rank[suc[off[mine[i]]:off[mine[i] + 1]]])
            assert np.array_equal(row, want)
        total += s.m
    assert total == int(off[-1])
    del states
    acc = hb.CentralityAccumulator(g.n)
    res = run_simulated(g, cfg, world, [acc])
    assert res.t == case["t"]
    for regs in res.registers:
        assert sha(regs) == case["reg_digests"][-1]


def test_packed_push_layout():
    """hb_push_row_stride: 12 bytes per row at p = 16 (25% below 16), 10 per 16 registers
    above (37.5% below p); wider registers fall back to the unpacked push."""
    from paper_1308_2144_b200 import _lib
    from paper_1308_2144_b200.distributed import CudaRankState, packed_push_stride
    L = _lib.hb()
    assert [L.hb_push_row_stride(b) for b in (4, 5, 6, 8, 12)] == [12, 20, 40, 160, 2560]
    assert L.hb_push_row_stride(3) == -1
    g = hb.CsrGraph.from_edges(np.arange(9), np.arange(1, 10), n=10)
    for width, want in ((5, 40), (6, 0)):
        cfg = hb.HyperBallConfig(params=hb.CounterParams(b=6, register_width=width))
        assert packed_push_stride(CudaRankState(g, cfg, 2, 0)) == want


def test_packed_push_wide_registers_unpacked():
    """register_width 6 (registers up to 59 need 6 bits): the push stays unpacked and the
    run is still bit-identical to one device."""
    case = CASES["rmat12_b7_s42_w5"]
    off, suc = golden_graph(case)
    g = hb.CsrGraph(off, suc)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=7, seed=3, register_width=6),
                             schedule="degree")
    a1 = hb.CentralityAccumulator(g.n)
    st = hb.run(g, cfg, [a1])
    a2 = hb.CentralityAccumulator(g.n)
    res = run_simulated(g, cfg, 3, [a2], exchange="push")
    assert res.t == st.t
    for regs in res.registers:
        assert sha(regs) == sha(st.register_matrix())
    assert np.array_equal(hb.finalize_harmonic(a1).view(np.uint64),
                          hb.finalize_harmonic(a2).view(np.uint64))
