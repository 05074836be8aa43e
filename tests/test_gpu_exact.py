"""The exact bitset backend on the GPU (engine.py:178-213, _kernels.py:117-172;
SURVEY.md 8(f) row 4): per-iteration bitset rows, estimates, sums and centralities must
equal the reference's exact runs bit for bit (tests/golden/ exact_cases), and the CPU
oracle's restatement on larger graphs."""

import hashlib

import numpy as np
import pytest

import oracle as orc
from conftest import exact_cases, golden, golden_graph

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_1308_2144_b200")
from paper_1308_2144_b200 import generators as gen  # noqa: E402

EXACT = exact_cases()


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bits_equal(a, b):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def _specs(case):
    return [hb.DiscountSpec.preset(name) if tab is None
            else hb.DiscountSpec.from_table(tab[0], tab[1], name="table")
            for name, tab in case.get("discounts") or []]


def drive(off, suc, weights=None, skip=True, specs=()):
    g = hb.CsrGraph(off, suc)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=6, seed=42), backend="exact",
                             weights=weights, skip_stable_nodes=skip)
    acc = hb.CentralityAccumulator(g.n, specs)
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


@pytest.mark.parametrize("skip", [True, False])
@pytest.mark.parametrize("case", EXACT, ids=[c["key"] for c in EXACT])
def test_exact_golden_case(case, skip):
    off, suc = golden_graph(case)
    _, arrays = golden()
    key = case["key"]
    w = arrays[f"{key}/weights"] if case.get("weights_seed") is not None else None
    specs = _specs(case)
    st, acc, regs, ests, nchs = drive(off, suc, w, skip, specs)
    assert st.t == case["t"]
    assert nchs == case["nch"]
    assert regs == case["reg_digests"]
    assert ests == case["est_digests"]
    fin = dict(sum_dist=acc.sum_dist, sum_recip=acc.sum_recip, coreach=acc.coreach,
               closeness=hb.finalize_closeness(acc), harmonic=hb.finalize_harmonic(acc),
               lin=hb.finalize_lin(acc))
    for spec in specs:
        fin[f"disc_{spec.name}"] = hb.finalize_discounted(acc, spec.name)
    for name, got in fin.items():
        assert bits_equal(got, arrays[f"{key}/{name}"]), name
    if specs and st.n:
        assert acc._binding is not None     # discounts fused into the exact kernel


def test_exact_checkpoint_bytes_match_reference(pins, tmp_path):
    p_, arrays = pins
    case = next(c for c in EXACT if c["key"] == "exact_islands400_nw2")
    off, suc = golden_graph(case)
    w = arrays["exact_islands400_nw2/weights"]
    g = hb.CsrGraph(off, suc)
    st = hb.initialize(g, hb.HyperBallConfig(params=hb.CounterParams(b=6, seed=42),
                                             weights=w, backend="exact"))
    hb.iterate(g, st)
    hb.iterate(g, st)
    path = tmp_path / "ck.bin"
    st.save(path)
    assert hashlib.sha256(path.read_bytes()).hexdigest() == p_["hbck_exact_islands400_nw2_t2"]
    back = hb.load_state(path)
    assert back.config.backend == "exact" and back.t == 2
    assert np.array_equal(back.register_matrix(), st.register_matrix())
    hb.resume(g, back)
    assert back.t == case["t"]
    assert sha(back.register_matrix()) == case["reg_digests"][-1]
    assert sha(back.est) == case["est_digests"][-1]
    with pytest.raises(ValueError):          # kind 1 cannot resume as probabilistic
        hb.load_state(path, hb.HyperBallConfig())


@pytest.mark.parametrize("n,avg,seed", [(1001, 2.5, 1), (129, 6.0, 2), (4000, 1.3, 3)])
def test_exact_vs_oracle_random(n, avg, seed):
    """Row lengths that are not multiples of 8 or 16 bytes (padding), sparse tails."""
    rng = np.random.default_rng(seed)
    m = int(n * avg)
    g = hb.CsrGraph.from_edges(rng.integers(0, n, m), rng.integers(0, n, m), n=n)
    w = rng.integers(1, 9, n)
    for weights in (None, w):
        res = orc.run_exact_oracle(g.offsets, g.successors, weights=weights)
        st, acc, regs, ests, nchs = drive(g.offsets, g.successors, weights)
        assert st.t == res.t and nchs == res.nch
        assert regs == res.reg_digests and ests == res.est_digests
        assert bits_equal(acc.sum_dist, res.sum_dist)
        assert bits_equal(hb.finalize_lin(acc), res.lin)


def test_exact_vs_oracle_rmat12():
    g = gen.rmat_t(12, 16 << 12, seed=11)
    res = orc.run_exact_oracle(g.offsets, g.successors)
    st, acc, regs, ests, nchs = drive(g.offsets, g.successors)
    assert st.t == res.t and nchs == res.nch
    assert regs == res.reg_digests and ests == res.est_digests
    assert bits_equal(hb.finalize_harmonic(acc), res.harmonic)


def test_exact_ball_members_and_errors():
    s = np.arange(9)
    g = hb.CsrGraph.from_edges(s[1:], s[:-1], n=10)     # transpose of a path 0 -> ... -> 8
    st = hb.run(g, hb.HyperBallConfig(backend="exact"))
    assert list(st.ball_members(8)) == list(range(9))
    assert list(st.ball_members(0)) == [0]
    assert list(st.ball_members(9)) == [9]
    assert np.array_equal(st.est[:9], np.arange(1, 10, dtype=np.float64))
    with pytest.raises(ValueError):
        st.counters()
    assert st.register_matrix().shape == (10, 2)


def test_exact_close_to_probabilistic():
    """test_engine.py's cross-backend check: HLL estimates within 3 sigma of exact."""
    rng = np.random.default_rng(31)
    n, m = 400, 1200
    g = hb.CsrGraph.from_edges(rng.integers(0, n, m), rng.integers(0, n, m), n=n)
    exact = hb.run(g, hb.HyperBallConfig(backend="exact")).est
    prob = hb.run(g, hb.HyperBallConfig(params=hb.CounterParams(b=12, seed=31))).est
    within = np.abs(prob - exact) <= np.maximum(3 * 0.0162 * exact, 1.0)
    assert within.mean() >= 0.99


def test_exact_run_multi():
    case = next(c for c in EXACT if c["key"] == "exact_random300_nw1")
    off, suc = golden_graph(case)
    _, arrays = golden()
    w = arrays["exact_random300_nw1/weights"]
    g = hb.CsrGraph(off, suc)
    out = hb.run_multi(g, hb.HyperBallConfig(backend="exact", weights=w), runs=2)
    for st, acc in out:                     # seeds differ, exact results do not
        assert st.t == case["t"]
        assert bits_equal(hb.finalize_harmonic(acc), arrays["exact_random300_nw1/harmonic"])


@pytest.mark.parametrize("key", ["exact_random300_nw1", "exact_sparse2000", "exact_cycle5"])
def test_reference_protocol_exact_backend(key):
    """CudaExactBackend driven the way engine.py:362-399 drives _ExactBackend."""
    from paper_1308_2144_b200.reference_backend import CudaExactBackend
    case = next(c for c in EXACT if c["key"] == key)
    off, suc = golden_graph(case)
    _, arrays = golden()
    w = arrays[f"{key}/weights"] if case.get("weights_seed") is not None else None
    g = hb.CsrGraph(off, suc)
    n = g.n
    be = CudaExactBackend(n, hb.CounterParams(b=6, seed=42), w, g)
    est, new_est = np.zeros(n), np.zeros(n)
    be.seed(w, est)
    changed_prev, changed_now = np.ones(n, dtype=bool), np.zeros(n, dtype=bool)
    regs, ests, t = [sha(be.cur)], [sha(est)], 0
    while True:
        nch = be.union_range(0, n, g.offsets, g.successors, changed_prev, changed_now, est,
                             new_est, True)
        t += 1
        be.swap()
        est, new_est = new_est, est
        changed_prev, changed_now = changed_now, changed_prev
        regs.append(sha(be.cur))
        ests.append(sha(est))
        if nch == 0:
            break
    assert t == case["t"]
    assert regs == case["reg_digests"] and ests == case["est_digests"]
