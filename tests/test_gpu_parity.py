"""Parity of the CUDA path (through the C-ABI) with the reference, on the GPU.

Golden cases: per-iteration register / estimate digests, changed counts, iteration count
and final centralities must equal the reference's bit for bit (tests/golden/, produced by
running the reference).  Larger seeded graphs: compared with the CPU oracle iteration by
iteration.  Tolerance for the fp64 centralities: exact (0 ulp) -- stronger than the 1e-9
relative bound BASELINE.json allows.
"""

import hashlib
import io

import numpy as np
import pytest
import torch

import oracle as orc
from conftest import golden, golden_cases, golden_graph

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_1308_2144_b200")
from paper_1308_2144_b200 import generators as gen  # noqa: E402

CASES = golden_cases()


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bits_equal(a, b):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def drive(off, suc, b, seed, width=5, schedule="auto", skip=True, weights=None):
    g = hb.CsrGraph(off, suc)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=b, register_width=width, seed=seed),
                             schedule=schedule, skip_stable_nodes=skip, weights=weights)
    acc = hb.CentralityAccumulator(g.n)
    st = hb.initialize(g, cfg)
    regs, ests, nchs = [sha(st.register_matrix())], [sha(st.est)], []
    if g.n:
        while True:
            nch = hb.iterate(g, st, [acc])
            regs.append(sha(st.register_matrix()))
            ests.append(sha(st.est))
            nchs.append(nch)
            if nch == 0:
                break
    acc.on_converged(st.est)
    return st, acc, regs, ests, nchs


@pytest.mark.parametrize("schedule", ["auto", "identity", "degree", "window"])
@pytest.mark.parametrize("case", CASES, ids=[c["key"] for c in CASES])
def test_golden_case(case, schedule):
    off, suc = golden_graph(case)
    _, arrays = golden()
    w = arrays[f"{case['key']}/weights"] if case.get("weights_seed") is not None else None
    st, acc, regs, ests, nchs = drive(off, suc, case["b"], int(case["seed"]), case["width"],
                                      schedule, weights=w)
    assert st.t == case["t"]
    assert nchs == case["nch"]
    assert regs == case["reg_digests"]
    assert ests == case["est_digests"]
    _, arrays = golden()
    key = case["key"]
    fin = dict(sum_dist=acc.sum_dist, sum_recip=acc.sum_recip, coreach=acc.coreach,
               closeness=hb.finalize_closeness(acc), harmonic=hb.finalize_harmonic(acc),
               lin=hb.finalize_lin(acc))
    for name, got in fin.items():
        assert bits_equal(got, arrays[f"{key}/{name}"]), name


def test_run_api_matches_golden_config1():
    case = next(c for c in CASES if c["key"] == "config1_b6_s42_w5")
    off, suc = golden_graph(case)
    g = hb.CsrGraph(off, suc)
    acc = hb.CentralityAccumulator(g.n)
    prog = io.StringIO()
    st = hb.run(g, hb.HyperBallConfig(params=hb.CounterParams(b=6, seed=42), progress=prog),
                [acc])
    _, arrays = golden()
    assert st.t == case["t"]
    assert bits_equal(hb.finalize_harmonic(acc), arrays["config1_b6_s42_w5/harmonic"])
    assert bits_equal(hb.finalize_lin(acc), arrays["config1_b6_s42_w5/lin"])
    lines = prog.getvalue().strip().splitlines()
    assert len(lines) == case["t"] and lines[-1].startswith(f"t={case['t']} changed=0")


def test_skip_equals_naive_on_gpu():
    case = next(c for c in CASES if c["key"].startswith("disc14_b4"))
    off, suc = golden_graph(case)
    a = drive(off, suc, 4, 42, skip=True)
    b = drive(off, suc, 4, 42, skip=False)
    assert a[2] == b[2] and a[3] == b[3]


def _oracle_compare(gT, b, seed, schedule="auto", max_iters=None):
    off = np.asarray(gT.offsets, np.int64)
    suc = np.asarray(gT.successors, np.int64)
    ref = orc.run_oracle(off, suc, b, seed, workers=8, record=True)
    st, acc, regs, ests, nchs = drive(off, suc, b, seed, schedule=schedule)
    assert nchs == ref.nch
    assert regs == ref.reg_digests
    assert ests == ref.est_digests
    assert bits_equal(acc.sum_dist, ref.sum_dist)
    assert bits_equal(acc.sum_recip, ref.sum_recip)
    assert bits_equal(hb.finalize_lin(acc), ref.lin)


@pytest.mark.parametrize("b", [4, 5, 7, 8, 9, 10, 12])
def test_rmat_heavy_split_vs_oracle(b):
    """R-MAT scale 14 has in-degrees in the thousands: exercises heavy items."""
    g = gen.rmat_t(14, 16 << 14, seed=21)
    _oracle_compare(g, b, 42)


@pytest.mark.parametrize("schedule", ["identity", "degree", "window"])
def test_rmat16_both_schedules(schedule):
    g = gen.rmat_t(16, 16 << 16, seed=22)
    _oracle_compare(g, 4, 7, schedule)


def test_estimate_rows_pins(pins):
    from paper_1308_2144_b200 import _lib
    from paper_1308_2144_b200.hll import estimator_constants, lc_table
    p_, arrays = pins
    for bs in p_["estimate_rows"]:
        b = int(bs)
        rows = torch.from_numpy(arrays[f"est_rows/{b}/rows"]).cuda()
        want = arrays[f"est_rows/{b}/est"]
        out = torch.zeros(rows.shape[0], dtype=torch.float64, device="cuda")
        lc = torch.from_numpy(lc_table(1 << b)).cuda()
        a2, cut, _ = estimator_constants(1 << b)
        _lib.check(_lib.hb().hb_estimate_rows(rows.data_ptr(), 0, rows.shape[0], b, lc.data_ptr(),
                                              a2, cut, out.data_ptr(),
                                              torch.cuda.current_stream().cuda_stream), "est")
        assert bits_equal(out.cpu().numpy(), want), b


def test_device_hash_pins(pins):
    from paper_1308_2144_b200 import _lib
    p_, _ = pins
    items = np.array([int(x) for x in p_["hash_items"]["items"]], dtype=np.uint64)
    for key, vals in p_["hash_items"]["values"].items():
        seed, replica = (int(x) for x in key.split(":"))
        it = torch.from_numpy(items.view(np.int64)).cuda()
        rp = torch.full_like(it, replica if replica < 2**63 else replica - 2**64)
        out = torch.empty_like(it)
        _lib.check(_lib.hb().hb_hash_items(it.numel(), it.data_ptr(), rp.data_ptr(), seed,
                                           out.data_ptr(), torch.cuda.current_stream().cuda_stream),
                   "hash")
        assert [str(int(h)) for h in out.cpu().numpy().view(np.uint64)] == vals


def test_checkpoint_bytes_match_reference(pins, tmp_path):
    p_, arrays = pins
    case = next(c for c in CASES if c["key"] == "random300_b6_s42_w5")
    off, suc = golden_graph(case)
    g = hb.CsrGraph(off, suc)
    st = hb.initialize(g, hb.HyperBallConfig(params=hb.CounterParams(b=6, seed=42)))
    hb.iterate(g, st)
    hb.iterate(g, st)
    path = tmp_path / "ck.bin"
    st.save(path)
    assert hashlib.sha256(path.read_bytes()).hexdigest() == p_["hbck_random300_b6_t2"]
    # resume from the checkpoint reaches the golden end state
    st2 = hb.load_state(path)
    hb.resume(g, st2)
    assert st2.t == case["t"]
    assert sha(st2.register_matrix()) == case["reg_digests"][-1]
    assert sha(st2.est) == case["est_digests"][-1]


@pytest.mark.parametrize("scale,factor,seed", [(10, 8, 3), (14, 16, 21), (16, 16, 22)])
def test_device_rmat_builder_matches_host(scale, factor, seed):
    """GPU graph build (hb_gen_rmat_keys + hb_keys_to_csr) == host C builder, byte for byte."""
    host = gen.rmat_t(scale, factor << scale, seed=seed)
    dev = gen.rmat_t_device(scale, factor << scale, seed=seed)
    assert dev.n == host.n and dev.m == host.m
    assert np.array_equal(dev.offsets.cpu().numpy(), host.offsets)
    assert np.array_equal(dev.successors.cpu().numpy(), host.successors)


def test_engine_on_device_graph():
    g = gen.rmat_t_device(12, 16 << 12, seed=11)
    case = next(c for c in CASES if c["key"] == "rmat12_b7_s42_w5")
    acc = hb.CentralityAccumulator(g.n)
    st = hb.run(g, hb.HyperBallConfig(params=hb.CounterParams(b=7, seed=42)), [acc])
    assert st.t == case["t"]
    assert sha(st.register_matrix()) == case["reg_digests"][-1]


def _specs(case):
    out = []
    for name, tab in case["discounts"]:
        out.append(hb.DiscountSpec.preset(name) if tab is None
                   else hb.DiscountSpec.from_table(tab[0], tab[1], name="table"))
    return out


@pytest.mark.parametrize("key", [c["key"] for c in CASES if c.get("discounts")])
def test_fused_discounts_match_reference(key):
    case = next(c for c in CASES if c["key"] == key)
    off, suc = golden_graph(case)
    g = hb.CsrGraph(off, suc)
    specs = _specs(case)
    acc = hb.CentralityAccumulator(g.n, specs)
    st = hb.run(g, hb.HyperBallConfig(params=hb.CounterParams(b=case["b"],
                                                             seed=int(case["seed"]))), [acc])
    assert acc._binding is not None        # fused on the device, not the host observer path
    assert st.t == case["t"]
    _, arrays = golden()
    for spec in specs:
        got = hb.finalize_discounted(acc, spec.name)
        want = arrays[f"{key}/disc_{spec.name}"]
        assert bits_equal(got, want), spec.name
    assert bits_equal(hb.finalize_harmonic(acc), arrays[f"{key}/harmonic"])


def test_run_multi_matches_independent_runs():
    """cli.py:222-254 repeated runs: run r uses seed + r; every run must equal an
    independent run (golden for r = 0, the oracle for r = 1, 2)."""
    case = next(c for c in CASES if c["key"] == "config1_b6_s42_w5")
    off, suc = golden_graph(case)
    g = hb.CsrGraph(off, suc)
    res = hb.run_multi(g, hb.HyperBallConfig(params=hb.CounterParams(b=6, seed=42)), runs=3)
    _, arrays = golden()
    assert res[0][0].t == case["t"]
    assert bits_equal(hb.finalize_harmonic(res[0][1]), arrays["config1_b6_s42_w5/harmonic"])
    for r in (1, 2):
        ref = orc.run_oracle(off, suc, 6, 42 + r, workers=4)
        assert res[r][0].t == ref.t
        assert bits_equal(hb.finalize_harmonic(res[r][1]), ref.harmonic)
        assert bits_equal(hb.finalize_lin(res[r][1]), ref.lin)
    mean, std = hb.multi_run_aggregate([hb.finalize_harmonic(a) for _, a in res])
    stack = np.vstack([hb.finalize_harmonic(a) for _, a in res])
    assert bits_equal(mean, stack.mean(axis=0)) and bits_equal(std, stack.std(axis=0, ddof=1))


@pytest.mark.parametrize("mode", ["forward", "pull", "pull-filtered", "off"])
@pytest.mark.parametrize("key", ["sparse2000_b4_s42_w5", "disc14_b4_s42_w5", "rmat12_b7_s42_w5",
                                 "islands400_b11_s3_w5", "config1_b6_s42_w5", "web14_b8_s42_w5"])
def test_frontier_mode_matches_reference(key, mode, monkeypatch):
    """Sparse iterations visiting only chg_prev | out-neighbours(chg_prev) give the
    reference's bits; the frontier is used whenever fewer than n counters changed, marked
    from the forward graph (hb_mark_active, 'forward') or by the pull pass over G^T
    (hb_mark_pull, 'pull'; with the shared-memory change filter, hb_mark_pull_filtered,
    'pull-filtered'); 'off' never."""
    from paper_1308_2144_b200 import engine as E
    monkeypatch.setattr(E, "FRONTIER_DIV", 1)
    monkeypatch.setattr(E, "FRONTIER_AFTER", 0 if mode == "forward" else 10**9)
    monkeypatch.setattr(E, "FILTER_MAX_CHANGED", 10**12 if mode == "pull-filtered" else -1)
    case = next(c for c in CASES if c["key"] == key)
    off, suc = golden_graph(case)
    g = hb.CsrGraph(off, suc)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=case["b"], seed=int(case["seed"])),
                             frontier=(mode != "off"))
    acc = hb.CentralityAccumulator(g.n)
    st = hb.initialize(g, cfg)
    regs, merged = [], []
    while True:
        nch = hb.iterate(g, st, [acc])
        regs.append(sha(st.register_matrix()))
        merged.append(st._dev.last_merged)
        if nch == 0:
            break
    acc.on_converged(st.est)
    assert st.t == case["t"]
    assert regs == case["reg_digests"][1:]
    _, arrays = golden()
    assert bits_equal(hb.finalize_lin(acc), arrays[f"{key}/lin"])
    if mode == "forward":
        assert st._dev.fwd is not None
    if mode.startswith("pull"):
        assert st._dev.fwd is None and st._dev.active is not None
        assert (st._dev.change_filter is not None) == (mode == "pull-filtered")


@pytest.mark.parametrize("key", ["random300_b6_s42_w5", "rmat12_b7_s42_w5", "sparse2000_b4_s42_w5"])
@pytest.mark.parametrize("schedule", ["identity", "degree"])
def test_reference_protocol_backend(key, schedule):
    """CudaBackend driven exactly like the reference engine drives its backends
    (engine.py:362-399: seed, union_range over [0, n), observers on host arrays, swap)."""
    from paper_1308_2144_b200.reference_backend import CudaBackend
    case = next(c for c in CASES if c["key"] == key)
    off, suc = golden_graph(case)
    g = hb.CsrGraph(off, suc)
    n = g.n
    params = hb.CounterParams(b=case["b"], seed=int(case["seed"]))
    be = CudaBackend(n, params, g, schedule=schedule)
    est = np.zeros(n)
    new_est = np.zeros(n)
    be.seed(None, est)
    changed_prev = np.ones(n, dtype=bool)
    changed_now = np.zeros(n, dtype=bool)
    acc = hb.CentralityAccumulator(n)
    regs = [sha(be.register_matrix())]
    ests = [sha(est)]
    t = 0
    while True:
        nch = be.union_range(0, n, g.offsets, g.successors, changed_prev, changed_now, est,
                             new_est, True)
        t += 1
        acc.on_step(t, est, new_est)          # host observer path, exactly as the reference
        be.swap()
        est, new_est = new_est, est
        changed_prev, changed_now = changed_now, changed_prev
        regs.append(sha(be.register_matrix()))
        ests.append(sha(est))
        if nch == 0:
            break
    acc.on_converged(est)
    assert t == case["t"]
    assert regs == case["reg_digests"] and ests == case["est_digests"]
    _, arrays = golden()
    assert bits_equal(hb.finalize_lin(acc), arrays[f"{key}/lin"])


def test_sorted_rows_schedule(monkeypatch):
    """HB_SORT_ROWS=1: degree relabel + per-row sort (hb_sort_rows) keeps the bits; rows
    come out ascending; multi-batch sorting (batches < 2^31 arcs) equals a host sort."""
    import ctypes
    from paper_1308_2144_b200 import _lib, schedule as S
    monkeypatch.setattr(S, "SORT_ROWS", True)
    case = next(c for c in CASES if c["key"] == "rmat12_b7_s42_w5")
    off, suc = golden_graph(case)
    g = hb.CsrGraph(off, suc)
    st = hb.run(g, hb.HyperBallConfig(params=hb.CounterParams(b=7, seed=42), schedule="degree"))
    assert st.t == case["t"] and sha(st.register_matrix()) == case["reg_digests"][-1]
    s = st._dev.sched
    o, v = s.offsets.cpu().numpy(), s.succ.cpu().numpy()
    assert all(np.all(np.diff(v[o[i]:o[i + 1]]) > 0) for i in range(s.n))
    # several batches
    rng = np.random.default_rng(5)
    deg = rng.integers(0, 40, 3000)
    offs = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    ids = rng.integers(0, 3000, int(offs[-1])).astype(np.int32)
    d_off = torch.from_numpy(offs).cuda()
    d_ids = torch.from_numpy(ids).cuda()
    alt = torch.empty_like(d_ids)
    br, ba = S._row_batches(d_off, 3000, int(offs[-1]), limit=7000)
    assert br.size > 3
    tb = ctypes.c_uint64(0)
    L = _lib.hb()
    args = (3000, d_off.data_ptr(), br.size - 1, br.ctypes.data_as(ctypes.c_void_p),
            ba.ctypes.data_as(ctypes.c_void_p), d_ids.data_ptr(), alt.data_ptr())
    _lib.check(L.hb_sort_rows(*args, None, ctypes.byref(tb), None, None), "size")
    temp = torch.empty(max(int(tb.value), 1), dtype=torch.uint8, device="cuda")
    _lib.check(L.hb_sort_rows(*args, temp.data_ptr(), ctypes.byref(tb), None, None), "sort")
    torch.cuda.synchronize()
    got = d_ids.cpu().numpy()
    want = np.concatenate([np.sort(ids[offs[i]:offs[i + 1]]) for i in range(3000)])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("b,width", [(4, 5), (5, 3), (6, 6), (7, 8), (8, 5), (12, 5), (4, 1)])
def test_device_register_packing(b, width):
    """hb_pack_registers / hb_unpack_registers == hll.pack_rows / unpack_rows (the HLLA
    layout, hll.py:145-177), with and without a row order."""
    from paper_1308_2144_b200 import _lib
    from paper_1308_2144_b200.hll import pack_rows, unpack_rows
    rng = np.random.default_rng(b * 10 + width)
    n, p = 1000, 1 << b
    regs = rng.integers(0, 1 << width, (n, p)).astype(np.uint8)
    order = rng.permutation(n).astype(np.int32)
    L = _lib.hb()
    d_regs = torch.from_numpy(regs).cuda()
    d_ord = torch.from_numpy(order).cuda()
    rb = p * width // 8
    for o in (None, d_ord):
        out = torch.empty((n, rb), dtype=torch.uint8, device="cuda")
        _lib.check(L.hb_pack_registers(n, b, width, d_regs.data_ptr(),
                                       o.data_ptr() if o is not None else None,
                                       out.data_ptr(), None), "pack")
        want = pack_rows(regs if o is None else regs[order], width)
        assert np.array_equal(out.cpu().numpy(), want)
        back = torch.empty_like(d_regs)
        _lib.check(L.hb_unpack_registers(n, b, width, out.data_ptr(),
                                         o.data_ptr() if o is not None else None,
                                         back.data_ptr(), None), "unpack")
        # unpack with the same order array: row i <- packed row order[i]
        exp = unpack_rows(want, p, width)
        exp = exp if o is None else exp[order]
        assert np.array_equal(back.cpu().numpy(), exp)
