"""The reference's OWN engine driving the B200 backend.

The reference package is imported from ``baseline/_ref`` (the one offline install of
``/root/reference/pkg``, git-ignored, shipped to the GPU box with the repo snapshot) and
its ``_ProbabilisticBackend`` is replaced by ``CudaBackend`` -- the registration a
maintainer would add at engine.py:342-345.  Everything else is the reference's code:
``initialize`` / ``iterate`` / ``run`` with its arc-balanced worker ranges on a thread
pool (engine.py:351-399), its HyperBallState, its CentralityAccumulator and finalizers.
Results must equal the golden digests the reference produced with its numba kernels, for
any worker count (test_engine.py:231-239).  Skipped where the package is not installed.
"""

import hashlib
import os
import sys

import numpy as np
import pytest

from conftest import REPO, golden, golden_cases, golden_graph

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_1308_2144_b200")


def _reference():
    path = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "hyperball")):
        pytest.skip("reference package not installed in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_hb")
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import hyperball
        from hyperball import engine as ref_engine
    except Exception as exc:  # numba missing etc.
        pytest.skip(f"reference package not importable: {exc!r}")
    return hyperball, ref_engine


CASES = {c["key"]: c for c in golden_cases()}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("workers", [1, 3, 8])
@pytest.mark.parametrize("schedule", ["auto", "identity", "degree"])
@pytest.mark.parametrize("key", ["random300_b6_s42_w5", "rmat12_b7_s42_w5",
                                 "sparse2000_b4_s42_w5", "config1_b6_s42_w5",
                                 "web14_b8_s42_w5"])
def test_reference_engine_with_cuda_backend(key, schedule, workers, monkeypatch):
    ref, ref_engine = _reference()
    from paper_1308_2144_b200.reference_backend import CudaBackend
    case = CASES[key]
    off, suc = golden_graph(case)
    g = ref.CsrGraph(np.asarray(off, np.int64), np.asarray(suc, np.int64))
    made = []

    def factory(n, params):
        be = CudaBackend(n, params, schedule=schedule)
        made.append(be)
        return be
    monkeypatch.setattr(ref_engine, "_ProbabilisticBackend", factory)
    cfg = ref.HyperBallConfig(params=ref.CounterParams(b=case["b"], seed=int(case["seed"])),
                              workers=workers)
    acc = ref.CentralityAccumulator(g.n)
    st = ref.initialize(g, cfg)
    assert made and st.backend is made[0]
    regs = [sha(st.register_matrix())]
    ests = [sha(st.est)]
    changed = []
    while True:
        nch = ref.iterate(g, st, [acc])
        changed.append(int(nch))
        regs.append(sha(st.register_matrix()))
        ests.append(sha(st.est))
        if nch == 0:
            break
    acc.on_converged(st.est)
    assert st.t == case["t"]
    assert regs == case["reg_digests"]
    assert ests == case["est_digests"]
    assert changed == case["nch"]
    _, arrays = golden()
    for name, fn in (("harmonic", ref.finalize_harmonic), ("closeness", ref.finalize_closeness),
                     ("lin", ref.finalize_lin)):
        got = fn(acc)
        assert np.array_equal(np.asarray(got).view(np.uint64),
                              arrays[f"{key}/{name}"].view(np.uint64)), name
    # the backend ran the device path: one full step per iteration, not one per worker
    assert made[0].t == st.t


@pytest.mark.parametrize("workers", [1, 4])
def test_reference_run_and_checkpoint_with_cuda_backend(workers, monkeypatch, tmp_path):
    """ref.run (engine.py:402-435) end to end, then the reference's own checkpoint writer
    (engine.py:254-280, counters() through the backend) reproduces the golden HBCK bytes
    when the golden case has one."""
    ref, ref_engine = _reference()
    from paper_1308_2144_b200.reference_backend import CudaBackend
    case = CASES["rmat12_b7_s42_w5"]
    off, suc = golden_graph(case)
    g = ref.CsrGraph(np.asarray(off, np.int64), np.asarray(suc, np.int64))
    monkeypatch.setattr(ref_engine, "_ProbabilisticBackend",
                        lambda n, params: CudaBackend(n, params))
    cfg = ref.HyperBallConfig(params=ref.CounterParams(b=case["b"], seed=int(case["seed"])),
                              workers=workers)
    acc = ref.CentralityAccumulator(g.n)
    st = ref.run(g, cfg, [acc])
    assert st.t == case["t"]
    assert sha(st.register_matrix()) == case["reg_digests"][-1]
    _, arrays = golden()
    assert np.array_equal(ref.finalize_harmonic(acc).view(np.uint64),
                          arrays["rmat12_b7_s42_w5/harmonic"].view(np.uint64))
    # packed counters through the backend equal the reference's own packing of the rows
    blob = st.counters().to_blob()
    dense = ref.CounterArray.from_dense(np.ascontiguousarray(st.register_matrix()),
                                        cfg.params).to_blob()
    assert blob == dense
