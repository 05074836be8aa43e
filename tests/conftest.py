"""Shared fixtures: the golden cases produced from the reference (tests/golden/) and the
graphs they were computed on."""

import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

GOLDEN_DIR = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


_golden = None


def golden():
    global _golden
    if _golden is None:
        with open(os.path.join(GOLDEN_DIR, "cases.json")) as fh:
            meta = json.load(fh)
        arrays = np.load(os.path.join(GOLDEN_DIR, "arrays.npz"))
        _golden = (meta, {k: arrays[k] for k in arrays.files})
    return _golden


_GEN_GRAPHS = {}


def golden_graph(case):
    """(offsets int64, successors int64) of the transpose graph a golden case ran on."""
    _, arrays = golden()
    name = case["graph"]
    if case["graph_stored"]:
        return arrays[f"graph/{name}/offsets"], arrays[f"graph/{name}/successors"]
    if name not in _GEN_GRAPHS:
        from paper_1308_2144_b200 import generators as gen
        builders = {
            "config1": lambda: gen.BUILDERS["config1"](),
            "config1_b4": lambda: gen.BUILDERS["config1"](),
            "rmat12": lambda: gen.rmat_t(12, 16 << 12, seed=11),
            "disc14": lambda: gen.disconnected_t(1 << 14, 1 << 13, 0.1, 6.0, seed=12),
            "web14": lambda: gen.weblike_t(1 << 14, seed=13, window=64),
        }
        g = builders[name]()
        assert gen.graph_digest(g) == case["graph_digest"], f"generator drift for {name}"
        _GEN_GRAPHS[name] = (np.asarray(g.offsets, np.int64), np.asarray(g.successors, np.int64))
    return _GEN_GRAPHS[name]


def golden_cases():
    meta, _ = golden()
    return meta["cases"]


def exact_cases():
    """Golden runs of the reference's exact bitset backend (engine.py:178-213)."""
    meta, _ = golden()
    return meta["exact_cases"]


@pytest.fixture(scope="session")
def pins():
    meta, arrays = golden()
    return meta["pins"], arrays
