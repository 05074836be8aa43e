"""Pin the CPU oracle (oracle/hb_oracle.c) to the reference's own outputs.

Every golden case was produced by running the reference package (tests/golden/
make_golden.py); the oracle must reproduce the per-iteration register and estimate
digests, the changed counts, the iteration count and the final centralities bit for bit.
"""

import hashlib

import numpy as np
import pytest

import oracle as orc
from conftest import exact_cases, golden, golden_cases, golden_graph

CASES = golden_cases()


@pytest.mark.parametrize("case", CASES, ids=[c["key"] for c in CASES])
def test_oracle_matches_reference(case):
    off, suc = golden_graph(case)
    _, arrays = golden()
    w = arrays[f"{case['key']}/weights"] if case.get("weights_seed") is not None else None
    res = orc.run_oracle(off, suc, case["b"], int(case["seed"]), case["width"], workers=2,
                         weights=w)
    assert res.t == case["t"]
    assert res.nch == case["nch"]
    assert res.reg_digests == case["reg_digests"]
    assert res.est_digests == case["est_digests"]
    _, arrays = golden()
    key = case["key"]
    for name in ("sum_dist", "sum_recip", "coreach", "closeness", "harmonic", "lin"):
        got = getattr(res, name)
        want = arrays[f"{key}/{name}"]
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), name


def test_oracle_skip_equals_naive():
    """skip_stable_nodes on/off give identical bits (test_engine.py:198-215)."""
    case = next(c for c in CASES if c["key"].startswith("sparse2000_b4"))
    off, suc = golden_graph(case)
    a = orc.run_oracle(off, suc, 4, 42, skip=True)
    b = orc.run_oracle(off, suc, 4, 42, skip=False)
    assert a.reg_digests == b.reg_digests and a.est_digests == b.est_digests


@pytest.mark.parametrize("workers", [1, 3, 8])
def test_oracle_worker_invariance(workers):
    case = next(c for c in CASES if c["key"].startswith("rmat12_b7"))
    off, suc = golden_graph(case)
    res = orc.run_oracle(off, suc, 7, 42, workers=workers)
    assert res.reg_digests == case["reg_digests"]


def test_hash_pins(pins):
    p, _ = pins
    items = np.array([int(x) for x in p["hash_items"]["items"]], dtype=np.uint64)
    for key, vals in p["hash_items"]["values"].items():
        seed, replica = (int(x) for x in key.split(":"))
        got = orc.hash_items(items, replica, seed)
        assert [str(int(h)) for h in got] == vals, key


def test_estimate_row_pins(pins):
    p, arrays = pins
    for b in p["estimate_rows"]:
        rows = arrays[f"est_rows/{b}/rows"]
        want = arrays[f"est_rows/{b}/est"]
        got = orc.estimate_rows(rows, int(b))
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), b


def test_alpha_pins(pins):
    p, _ = pins
    for ps, a2 in p["alpha_p2"].items():
        assert orc.constants(int(ps).bit_length() - 1)[0] == a2


EXACT = exact_cases()


@pytest.mark.parametrize("case", EXACT, ids=[c["key"] for c in EXACT])
def test_exact_oracle_matches_reference(case):
    """The exact-backend restatement (oracle.run_exact_oracle) reproduces the reference's
    exact runs: per-iteration bitset rows, estimates, sums and centralities."""
    off, suc = golden_graph(case)
    _, arrays = golden()
    key = case["key"]
    w = arrays[f"{key}/weights"] if case.get("weights_seed") is not None else None
    res = orc.run_exact_oracle(off, suc, weights=w)
    assert res.t == case["t"]
    assert res.nch == case["nch"]
    assert res.reg_digests == case["reg_digests"]
    assert res.est_digests == case["est_digests"]
    for name in ("sum_dist", "sum_recip", "coreach", "closeness", "harmonic", "lin"):
        got = getattr(res, name)
        assert np.array_equal(got.view(np.uint64), arrays[f"{key}/{name}"].view(np.uint64)), name


def test_exact_oracle_skip_equals_naive():
    case = next(c for c in EXACT if c["key"] == "exact_sparse2000")
    off, suc = golden_graph(case)
    a = orc.run_exact_oracle(off, suc, skip=True)
    b = orc.run_exact_oracle(off, suc, skip=False)
    assert a.reg_digests == b.reg_digests and a.est_digests == b.est_digests


@pytest.mark.parametrize("name", ["config1", "config2", "config3"])
def test_oracle_matches_reference_at_full_size(name):
    """The oracle against the reference's own full-size runs (tests/golden/fullsize.json,
    tests/golden/make_fullsize.py): registers and estimates after every iteration,
    changed counts, t and the finalizers, on BASELINE.json's configs 1-3 (config 4 is
    pinned on the GPU box, where the device run is compared with the same fixture)."""
    import json
    import os
    import sys

    from conftest import GOLDEN_DIR
    sys.path.insert(0, GOLDEN_DIR)
    from digest import reg_digest
    from paper_1308_2144_b200 import generators as gen

    want = json.load(open(os.path.join(GOLDEN_DIR, "fullsize.json")))[name]
    cfgd = gen.CONFIGS[name]
    g = cfgd.build()
    assert gen.graph_digest(g) == want["graph_digest"]
    res = orc.run_oracle(np.asarray(g.offsets, np.int64), np.asarray(g.successors, np.int64),
                         cfgd.log2m, cfgd.hash_seed, 5, workers=os.cpu_count() or 1,
                         reg_digest=reg_digest)
    assert res.t == want["t"]
    assert res.nch == want["nch"]
    assert res.reg_digests == want["reg_digests"]
    assert res.est_digests == want["est_digests"]
    for nm in ("closeness", "harmonic", "lin"):
        assert hashlib.sha256(getattr(res, nm).tobytes()).hexdigest() == want[nm], nm
