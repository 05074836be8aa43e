"""Engine behaviour on the GPU, mirroring the reference's tests/test_engine.py for the
probabilistic backend (initialize / iterate / run / resume semantics, observers,
errors, progress lines, register monotonicity, schedule invariance, checkpoints)."""

import io
from collections import deque

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_1308_2144_b200")
from paper_1308_2144_b200.hll import CounterArray  # noqa: E402


def cfg(b=12, seed=0, **kw):
    return hb.HyperBallConfig(params=hb.CounterParams(b=b, seed=seed), **kw)


def path_graph(k):
    s = np.arange(k - 1)
    return hb.CsrGraph.from_edges(s, s + 1, n=k)


def cycle_graph(k):
    s = np.arange(k)
    return hb.CsrGraph.from_edges(s, (s + 1) % k, n=k)


def star_graph(k):
    return hb.CsrGraph.from_edges(np.zeros(k, np.int64), np.arange(1, k + 1), n=k + 1)


def random_graph(seed, n, avg):
    rng = np.random.default_rng(seed)
    m = int(round(n * avg))
    return hb.CsrGraph.from_edges(rng.integers(0, n, m), rng.integers(0, n, m), n=n)


def bfs_sizes(g):
    """Forward-reachable set sizes by plain BFS (test_engine.py's low-tech reference)."""
    succ = [list(g.successors_of(v)) for v in range(g.n)]
    out = np.zeros(g.n)
    for s in range(g.n):
        seen = {s}
        q = deque([s])
        while q:
            v = q.popleft()
            for w in succ[v]:
                if w not in seen:
                    seen.add(w)
                    q.append(w)
        out[s] = len(seen)
    return out


class TestInitialize:
    def test_unweighted_estimates_one(self):
        st = hb.initialize(path_graph(4), cfg())
        assert np.all(np.abs(st.est - 1.0) < 0.01)

    def test_weighted_replicas(self):
        st = hb.initialize(path_graph(3), cfg(seed=2, weights=np.array([5, 1, 2])))
        assert abs(st.est[0] - 5.0) <= 3 * 0.0162 * 5.0

    def test_weight_validation(self):
        with pytest.raises(ValueError):
            hb.initialize(path_graph(3), cfg(weights=np.array([1, 0, 1])))
        with pytest.raises(ValueError):
            hb.initialize(path_graph(3), cfg(weights=np.ones(5, np.int64)))
        heavy = np.array([2**31, 2**31], np.int64)
        with pytest.raises(ValueError, match="register_width 6"):
            hb.initialize(path_graph(2), hb.HyperBallConfig(
                params=hb.CounterParams(b=4, register_width=5), weights=heavy))

    def test_empty_graph(self):
        g = hb.CsrGraph(np.zeros(1, np.int64), np.zeros(0, np.int64))
        st = hb.run(g, cfg())
        assert st.t == 0 and st.num_changed == 0


class TestIterate:
    def test_no_arcs_converges_immediately(self):
        g = hb.CsrGraph.from_edges([], [], n=6)
        st = hb.initialize(g, cfg())
        assert hb.iterate(g, st) == 0

    def test_star_two_iterations(self):
        st = hb.run(star_graph(7), cfg())
        assert st.t == 2

    def test_cycle_five(self):
        st = hb.run(cycle_graph(5), cfg())
        assert st.t == 5

    def test_isolated_nodes_one_iteration(self):
        st = hb.run(hb.CsrGraph.from_edges([], [], n=9), cfg())
        assert st.t == 1

    def test_observer_contract(self):
        g = path_graph(3)
        st = hb.initialize(g, cfg())
        seen = []

        class Recorder:
            def on_step(self, t, old, new):
                seen.append((t, old.copy(), new.copy()))

            def on_converged(self, final):
                seen.append(("done", final.copy()))

        out = hb.resume(g, st, [Recorder()])
        assert out.t == 3
        t2 = seen[1]
        assert t2[0] == 2
        assert t2[1][2] == t2[2][2]          # node 2 (no successors) is stable
        assert seen[-1][0] == "done"
        assert np.array_equal(seen[-1][1], out.est)

    def test_probabilistic_close_to_exact(self):
        g = random_graph(31, 400, 3.0)
        exact = bfs_sizes(g)
        prob = hb.run(g, cfg(b=12, seed=31)).est
        within = np.abs(prob - exact) <= np.maximum(3 * 0.0162 * exact, 1.0)
        assert within.mean() >= 0.99

    def test_max_iterations_reports_state(self):
        with pytest.raises(hb.ConvergenceError) as err:
            hb.run(path_graph(50), cfg(max_iterations=3))
        assert err.value.t == 3 and err.value.num_changed > 0

    def test_progress_lines(self):
        stream = io.StringIO()
        hb.run(path_graph(4), cfg(progress=stream))
        lines = stream.getvalue().strip().splitlines()
        assert len(lines) == 4
        assert lines[0].startswith("t=1 changed=3 elapsed_ms=")


class TestRegisterSemantics:
    def test_register_monotonicity_over_run(self):
        g = random_graph(5, 60, 2.0)
        st = hb.initialize(g, cfg(b=4, seed=5))
        prev = st.register_matrix().copy()
        while True:
            changed = hb.iterate(g, st)
            cur = st.register_matrix()
            assert np.all(cur >= prev)
            prev = cur.copy()
            if changed == 0:
                break

    @pytest.mark.parametrize("b", [4, 6, 8])
    def test_schedule_invariance(self, b):
        """Worker-count invariance (test_engine.py:231-239) for the B200 schedules."""
        g = random_graph(7, 500, 3.0)
        outs = [hb.run(g, cfg(b=b, seed=9, schedule=s)) for s in ("identity", "degree", "window")]
        for o in outs[1:]:
            assert outs[0].t == o.t
            assert np.array_equal(outs[0].register_matrix(), o.register_matrix())
            assert np.array_equal(outs[0].est.view(np.uint64), o.est.view(np.uint64))

    def test_counters_pack_registers(self):
        g = random_graph(3, 100, 2.0)
        st = hb.run(g, cfg(b=6, seed=1))
        packed = st.counters()
        assert packed == CounterArray.from_dense(st.register_matrix(), st.config.params)
        assert np.array_equal(packed.to_dense(), st.register_matrix())

    def test_estimates_is_a_copy(self):
        st = hb.initialize(path_graph(5), cfg())
        a = st.estimates()
        a[:] = -1
        assert np.all(st.estimates() > 0)

    def test_register_matrix_read_only(self):
        st = hb.initialize(path_graph(5), cfg())
        with pytest.raises(ValueError):
            st.register_matrix()[0, 0] = 1


class TestCheckpoint:
    def test_roundtrip_midway(self, tmp_path):
        g = random_graph(11, 300, 2.0)
        full = hb.run(g, cfg(b=7, seed=4))
        st = hb.initialize(g, cfg(b=7, seed=4))
        hb.iterate(g, st)
        hb.iterate(g, st)
        path = tmp_path / "ck.bin"
        st.save(path)
        back = hb.load_state(path)
        assert back.t == 2
        assert np.array_equal(back.register_matrix(), st.register_matrix())
        hb.resume(g, back)
        assert back.t == full.t
        assert np.array_equal(back.register_matrix(), full.register_matrix())
        assert np.array_equal(back.est.view(np.uint64), full.est.view(np.uint64))


class TestLazyCoreach:
    """run() with only a fused accumulator keeps the final estimates on the device: the
    accumulator's coreach is downloaded on first read and equals the state's estimates."""

    def test_coreach_lazy_and_exact(self):
        g = random_graph(4, 3000, 5.0)
        acc = hb.CentralityAccumulator(g.n)
        st = hb.run(g, cfg(b=8, seed=3), [acc])
        assert acc.converged and acc._coreach_fetch is not None
        lin = hb.finalize_lin(acc)                    # on the device, no host coreach
        assert acc._coreach_fetch is not None
        c = acc.coreach
        assert acc._coreach_fetch is None and not c.flags.writeable
        assert np.array_equal(c.view(np.uint64), st.est.view(np.uint64))
        s = acc.sum_dist
        want = np.divide(c * c, s, out=np.ones_like(s), where=s > 0)
        assert np.array_equal(lin.view(np.uint64), want.view(np.uint64))

    def test_reassigned_coreach_goes_host_path(self):
        g = random_graph(5, 2000, 4.0)
        acc = hb.CentralityAccumulator(g.n)
        hb.run(g, cfg(b=6, seed=1), [acc])
        acc.coreach = np.full(g.n, 2.0)
        s = acc.sum_dist
        want = np.divide(4.0, s, out=np.ones_like(s), where=s > 0)
        assert np.array_equal(hb.finalize_lin(acc), want)

    def test_extra_observer_gets_host_copy(self):
        class Last(hb.BallObserver):
            final = None

            def on_converged(self, final_estimates):
                self.final = final_estimates
        g = random_graph(6, 2000, 4.0)
        acc, last = hb.CentralityAccumulator(g.n), Last()
        st = hb.run(g, cfg(b=6, seed=2), [acc, last])
        assert last.final is not None and acc._coreach_fetch is None
        assert np.array_equal(acc.coreach, st.est) and np.array_equal(last.final, st.est)


@pytest.mark.skipif(not __import__("torch").cuda.is_available()
                    or __import__("torch").cuda.device_count() < 2,
                    reason="needs two GPUs in one process")
def test_two_devices_in_one_process():
    """Per-device library state (SM count, opt-in shared memory of the p = 256 TMA kernel,
    L2 set-aside) and the stream-device guard: runs on devices 0 and 1 stepped
    alternately from one thread, with device 0 current throughout, give identical bits."""
    import torch
    torch.cuda.set_device(0)
    g = random_graph(5, 3000, 6.0)
    for b in (4, 8):
        states = [hb.initialize(g, cfg(b=b, seed=3, device=d)) for d in (0, 1)]
        accs = [hb.CentralityAccumulator(g.n) for _ in states]
        while True:
            nch = [hb.iterate(g, st, [a]) for st, a in zip(states, accs)]
            assert nch[0] == nch[1]
            assert np.array_equal(states[0].register_matrix(), states[1].register_matrix())
            if nch[0] == 0:
                break
        for a in accs:
            a.on_converged(states[accs.index(a)].est)
        for fin in (hb.finalize_harmonic, hb.finalize_lin):
            assert np.array_equal(fin(accs[0]).view(np.uint64), fin(accs[1]).view(np.uint64))
        assert torch.cuda.current_device() == 0
