"""Batched repeated runs (multirun.py, hb_union_step_runs): R seeds sharing one union pass
must give, run by run, the bits of independent runs -- registers, estimates, iteration
counts, accumulator sums and centralities -- and call the observers as the reference's
per-run loop does (cli.py:222-254, engine.py:413-435); every run is also checked against
the CPU oracle run with seed + r."""

import hashlib

import numpy as np
import pytest

from conftest import golden, golden_cases, golden_graph

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_1308_2144_b200")
from paper_1308_2144_b200 import multirun  # noqa: E402
import oracle as orc  # noqa: E402  (the checker; tests/conftest.py puts oracle/ on the path)

CASES = {c["key"]: c for c in golden_cases()}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


class Counter:
    def __init__(self):
        self.steps = []
        self.final = None

    def on_step(self, t, old, new):
        self.steps.append((t, sha(old), sha(new)))

    def on_converged(self, final):
        self.final = sha(final)


def _compare(g, cfg, runs, batch):
    ref_obs = {}
    got_obs = {}

    def f_ref(r):
        ref_obs[r] = Counter()
        return [ref_obs[r]]

    def f_got(r):
        got_obs[r] = Counter()
        return [got_obs[r]]
    ref = hb.run_multi(g, cfg, runs, observers_factory=f_ref, batch=1)
    got = hb.run_multi(g, cfg, runs, observers_factory=f_got, batch=batch)
    for r in range(runs):
        (sa, aa), (sb, ab) = ref[r], got[r]
        assert sb.t == sa.t, (r, sa.t, sb.t)
        assert sha(sb.register_matrix()) == sha(sa.register_matrix())
        assert np.array_equal(bits(sb.est), bits(sa.est))
        for fin in (hb.finalize_harmonic, hb.finalize_closeness, hb.finalize_lin):
            assert np.array_equal(bits(fin(ab)), bits(fin(aa))), fin.__name__
        assert got_obs[r].steps == ref_obs[r].steps
        assert got_obs[r].final == ref_obs[r].final
    # every run r also against the CPU oracle with seed + r (cli.py:222-254): iteration
    # count, final registers, estimates and the three centralities, bit for bit
    pr = cfg.params
    for r in range(runs):
        want = orc.run_oracle(np.asarray(g.offsets, np.int64), np.asarray(g.successors, np.int64),
                              pr.b, pr.seed + r, width=pr.register_width, workers=4,
                              skip=cfg.skip_stable_nodes,
                              weights=None if cfg.weights is None else
                              np.asarray(getattr(cfg.weights, "values", cfg.weights), np.int64))
        st, acc = got[r]
        assert st.t == want.t, (r, st.t, want.t)
        assert sha(st.register_matrix()) == want.reg_digests[-1], r
        assert np.array_equal(bits(st.est), bits(want.est)), r
        for fin, arr in ((hb.finalize_harmonic, want.harmonic),
                         (hb.finalize_closeness, want.closeness), (hb.finalize_lin, want.lin)):
            assert np.array_equal(bits(fin(acc)), bits(arr)), (r, fin.__name__)
    return got


@pytest.mark.parametrize("key,batch", [
    ("random300_b4_s42_w5", 2), ("random300_b4_s42_w5", 4), ("random300_b4_s42_w5", 8),
    ("random300_b4_s42_w5", 16), ("sparse2000_b4_s42_w5", 4), ("rmat12_b4_s42_w5", 4),
    ("rmat12_b4_s42_w5", 16), ("disc14_b4_s42_w5", 8), ("random300_b5_s42_w5", 2),
    ("random300_b5_s42_w5", 8), ("random300_b6_s42_w5", 4), ("random300_b7_s42_w5", 2),
    ("rmat12_b7_s42_w5", 2), ("islands400_b6_s3_w5", 4), ("config1_b6_s42_w5", 4),
    ("web14_b8_s42_w5", 1)])
def test_batched_runs_equal_independent_runs(key, batch):
    case = CASES[key]
    off, suc = golden_graph(case)
    g = hb.CsrGraph(off, suc)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=case["b"], seed=int(case["seed"])))
    got = _compare(g, cfg, max(batch, 2) + 1, batch)   # a ragged last group too
    # run 0 is the golden case itself
    st, acc = got[0]
    assert st.t == case["t"]
    assert sha(st.register_matrix()) == case["reg_digests"][-1]
    _, arrays = golden()
    assert np.array_equal(bits(hb.finalize_lin(acc)), bits(arrays[f"{key}/lin"]))


@pytest.mark.parametrize("schedule", ["identity", "degree", "window"])
def test_batched_runs_schedules(schedule):
    case = CASES["rmat12_b4_s42_w5"]
    off, suc = golden_graph(case)
    g = hb.CsrGraph(off, suc)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=4, seed=7), schedule=schedule)
    _compare(g, cfg, 4, 4)


def test_batched_weighted_and_naive():
    case = CASES["random300_b6_s42_w5_nw1"]
    off, suc = golden_graph(case)
    _, arrays = golden()
    w = arrays["random300_b6_s42_w5_nw1/weights"]
    g = hb.CsrGraph(off, suc)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=6, seed=42), weights=w)
    got = _compare(g, cfg, 4, 4)
    assert sha(got[0][0].register_matrix()) == case["reg_digests"][-1]
    cfg2 = hb.HyperBallConfig(params=hb.CounterParams(b=4, seed=3), skip_stable_nodes=False)
    _compare(g, cfg2, 4, 4)


@pytest.mark.parametrize("schedule", ["auto", "window"])
def test_batched_states_are_ordinary_states(tmp_path, schedule):
    """Returned states checkpoint, pack and keep iterating like run()'s (iterating builds
    the single-run schedule and carries the device sums over)."""
    case = CASES["sparse2000_b4_s42_w5"]
    off, suc = golden_graph(case)
    g = hb.CsrGraph(off, suc)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=4, seed=42), schedule=schedule)
    (st, acc), *_ = hb.run_multi(g, cfg, 4, batch=4)
    solo_acc = hb.CentralityAccumulator(g.n)
    solo = hb.run(g, cfg, [solo_acc])
    assert st.counters() == solo.counters()
    st.save(tmp_path / "a.bin")
    solo.save(tmp_path / "b.bin")
    assert (tmp_path / "a.bin").read_bytes() == (tmp_path / "b.bin").read_bytes()
    assert acc._binding is not None              # sums stayed on the device
    assert hb.iterate(g, st, [acc]) == 0
    assert hb.iterate(g, solo, [solo_acc]) == 0
    for fin in (hb.finalize_harmonic, hb.finalize_closeness):
        assert np.array_equal(bits(fin(acc)), bits(fin(solo_acc)))
    assert np.array_equal(bits(st.est), bits(solo.est))


def test_batched_max_iterations():
    s = np.arange(59)
    g = hb.CsrGraph.from_edges(s + 1, s, n=60)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=4, seed=1), max_iterations=5)
    with pytest.raises(hb.ConvergenceError):
        hb.run_multi(g, cfg, 4, batch=4)


def test_batch_size_policy():
    assert multirun.batch_size(16, 10) == 4 and multirun.batch_size(32, 10) == 2
    assert multirun.batch_size(64, 10) == 1 and multirun.batch_size(16, 1) == 1
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=4))
    assert multirun.supported(cfg, 4) and multirun.supported(cfg, 16)
    assert not multirun.supported(cfg, 3) and not multirun.supported(cfg, 32)


def test_batched_discounts_and_progress():
    """Fused discounts per run ([R, k, n] on the device) and the per-run progress lines of
    the reference loop (engine.py:420-425), written run after run."""
    import io
    import re
    case = CASES["random300_b4_s42_w5"]
    off, suc = golden_graph(case)
    g = hb.CsrGraph(off, suc)
    specs = [hb.DiscountSpec.preset("harmonic"), hb.DiscountSpec.preset("log"),
             hb.DiscountSpec.from_table((1.0, 0.5, 0.25), 0.125, name="table")]
    outs, prog = {}, {}
    for batch in (1, 4):
        prog[batch] = io.StringIO()
        cfg = hb.HyperBallConfig(params=hb.CounterParams(b=4, seed=42), progress=prog[batch])
        outs[batch] = hb.run_multi(g, cfg, 4, discounts=specs, batch=batch)
    for (sa, aa), (sb, ab) in zip(outs[1], outs[4]):
        assert sa.t == sb.t
        for spec in specs:
            assert np.array_equal(bits(hb.finalize_discounted(aa, spec.name)),
                                  bits(hb.finalize_discounted(ab, spec.name))), spec.name
        assert np.array_equal(bits(hb.finalize_harmonic(aa)), bits(hb.finalize_harmonic(ab)))
    strip = [re.sub(r"elapsed_ms=\d+", "", prog[b].getvalue()) for b in (1, 4)]
    assert strip[0] == strip[1] and strip[0].count("\n") == sum(s.t for s, _ in outs[1])
    assert outs[4][0][1]._binding is not None          # discounts stayed on the device
