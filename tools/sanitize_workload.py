"""Small workloads covering every kernel family, for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck):

    compute-sanitizer --tool memcheck python tools/sanitize_workload.py

* p = 256 light kernel with the TMA row gather + mbarrier (web-like graph, window order)
* p = 16 heavy items + finish + range-policy loads (R-MAT, degree order)
* frontier marking (pull, filtered, forward graph) in the sparse tail
* fused multi-GPU push and the all-gather exchange on simulated ranks
* batched runs, the exact backend, checkpoint pack / unpack, device graph builders,
  device transpose
Every result is checked against the CPU oracle, so a run that completes under the tool
also completed correctly.
"""
import hashlib
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

import oracle as orc  # noqa: E402
import paper_1308_2144_b200 as hb  # noqa: E402
from paper_1308_2144_b200 import generators as gen  # noqa: E402
from paper_1308_2144_b200.distributed import run_simulated  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def check_run(g, b, schedule, **kw):
    ref = orc.run_oracle(np.asarray(g.offsets, np.int64), np.asarray(g.successors, np.int64),
                         b, 42, workers=4)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=b, seed=42), schedule=schedule, **kw)
    acc = hb.CentralityAccumulator(g.n)
    st = hb.run(g, cfg, [acc])
    assert st.t == ref.t, (st.t, ref.t)
    assert sha(st.register_matrix()) == ref.reg_digests[-1]
    assert np.array_equal(hb.finalize_harmonic(acc).view(np.uint64), ref.harmonic.view(np.uint64))
    return st


def main():
    which = sys.argv[1:] or ["tma", "heavy", "frontier", "push", "allgather", "multi", "exact",
                             "ckpt", "build"]
    web = gen.weblike_t(1 << 13, seed=13, window=64)
    rmat = gen.rmat_t(12, 16 << 12, seed=11)
    if "tma" in which:
        check_run(web, 8, "window")
        check_run(web, 8, "identity")
        print("tma ok", flush=True)
    if "heavy" in which:
        check_run(rmat, 4, "degree")
        check_run(rmat, 7, "degree")
        print("heavy ok", flush=True)
    if "frontier" in which:
        d = gen.disconnected_t(1 << 13, 1 << 12, 0.1, 6.0, seed=12)
        check_run(d, 6, "identity")
        check_run(rmat, 5, "degree")
        print("frontier ok", flush=True)
    for ex in ("push", "allgather"):
        if ex in which:
            ref = orc.run_oracle(np.asarray(rmat.offsets, np.int64),
                                 np.asarray(rmat.successors, np.int64), 7, 42, workers=4)
            cfg = hb.HyperBallConfig(params=hb.CounterParams(b=7, seed=42), schedule="degree")
            res = run_simulated(rmat, cfg, 3, [hb.CentralityAccumulator(rmat.n)], exchange=ex)
            assert res.t == ref.t
            assert all(sha(r) == ref.reg_digests[-1] for r in res.registers)
            print(ex, "ok", flush=True)
    if "multi" in which:
        out = hb.run_multi(rmat, hb.HyperBallConfig(params=hb.CounterParams(b=4, seed=42)), 4)
        ref = orc.run_oracle(np.asarray(rmat.offsets, np.int64),
                             np.asarray(rmat.successors, np.int64), 4, 43, workers=4)
        assert sha(out[1][0].register_matrix()) == ref.reg_digests[-1]
        print("multi ok", flush=True)
    if "exact" in which:
        small = gen.rmat_t(9, 8 << 9, seed=3)
        st = hb.run(small, hb.HyperBallConfig(backend="exact"))
        ref = orc.run_exact_oracle(np.asarray(small.offsets, np.int64),
                                   np.asarray(small.successors, np.int64))
        assert st.t == ref.t
        print("exact ok", flush=True)
    if "ckpt" in which:
        import tempfile
        cfg = hb.HyperBallConfig(params=hb.CounterParams(b=6, seed=42))
        st = hb.initialize(rmat, cfg)
        hb.iterate(rmat, st)
        with tempfile.TemporaryDirectory() as td:
            st.save(os.path.join(td, "c.bin"))
            st2 = hb.load_state(os.path.join(td, "c.bin"), graph=rmat)
        assert sha(st2.register_matrix()) == sha(st.register_matrix())
        print("ckpt ok", flush=True)
    if "build" in which:
        for host, dev in ((lambda: gen.weblike_t(1 << 12, seed=4, window=64),
                           lambda: gen.weblike_t_device(1 << 12, seed=4, window=64)),
                          (lambda: gen.disconnected_t(4096, 1024, 0.2, 4.0, seed=2),
                           lambda: gen.disconnected_t_device(4096, 1024, 0.2, 4.0, seed=2)),
                          (lambda: gen.rmat_t(10, 8 << 10, seed=2),
                           lambda: gen.rmat_t_device(10, 8 << 10, seed=2))):
            assert gen.graph_digest(host()) == gen.graph_digest(dev().to_host())
        t = hb.transpose_device(rmat)
        assert np.array_equal(t.to_host().offsets, hb.transpose(rmat).offsets)
        print("build ok", flush=True)
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
