"""GPU graph build: the device builders of every synthetic config and
the device transpose, against the host builders and the reference's own outputs.

* hb_transpose_csr == the reference's transpose (graph.py:145-155) on the fixtures of
  tests/golden/make_transpose_golden.py (duplicates, self-loops, empty rows), from host
  and from device input.
* hb_gen_degrees / hb_gen_blocks / hb_gen_arc_keys + hb_keys_to_csr produce the host
  builder's bytes (graphgen.c) at small sizes, and at BASELINE.json's full sizes the graph
  digests recorded with the reference's full-size runs (tests/golden/fullsize.json).
* A device-built transpose feeds the engine: registers equal the host path's.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR, golden_cases, golden_graph

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_1308_2144_b200")
import torch  # noqa: E402

from paper_1308_2144_b200 import generators as gen  # noqa: E402


def _tgold():
    z = np.load(os.path.join(GOLDEN_DIR, "transpose.npz"))
    return z, [str(x) for x in z["names"]]


def _host(g):
    return (np.asarray(g.offsets.cpu() if isinstance(g.offsets, torch.Tensor) else g.offsets,
                       np.int64),
            np.asarray(g.successors.cpu() if isinstance(g.successors, torch.Tensor)
                       else g.successors, np.int64))


@pytest.mark.parametrize("on_device", [False, True])
def test_transpose_device_matches_reference(on_device):
    z, names = _tgold()
    for nm in names:
        off, suc = z[f"{nm}/offsets"], z[f"{nm}/successors"]
        if on_device:
            g = hb.DeviceCsrGraph(torch.from_numpy(off).cuda(),
                                  torch.from_numpy(suc.astype(np.int32)).cuda())
            t = hb.transpose(g)                  # a DeviceCsrGraph transposes on its device
        else:
            t = hb.transpose_device(hb.CsrGraph(off, suc))
        assert isinstance(t, hb.DeviceCsrGraph)
        o, s = _host(t)
        assert np.array_equal(o, z[f"{nm}/t_offsets"]), nm
        assert np.array_equal(s, z[f"{nm}/t_successors"]), nm


def test_transpose_device_is_an_involution_on_normalised_graphs():
    g = gen.rmat_t(12, 16 << 12, seed=11)          # normalised: sorted rows, no duplicates
    tt = hb.transpose_device(hb.transpose_device(g))
    o, s = _host(tt)
    assert np.array_equal(o, np.asarray(g.offsets, np.int64))
    assert np.array_equal(s, np.asarray(g.successors, np.int64))


SMALL = [
    ("er", lambda: gen.erdos_renyi_t(3000, 8.0, seed=5),
     lambda: gen.erdos_renyi_t_device(3000, 8.0, seed=5)),
    ("disc", lambda: gen.disconnected_t(1 << 14, 1 << 13, 0.1, 6.0, seed=12),
     lambda: gen.disconnected_t_device(1 << 14, 1 << 13, 0.1, 6.0, seed=12)),
    ("disc_small_giant", lambda: gen.disconnected_t(5000, 7, 0.3, 3.0, seed=1),
     lambda: gen.disconnected_t_device(5000, 7, 0.3, 3.0, seed=1)),
    ("web", lambda: gen.weblike_t(1 << 14, seed=13, window=64),
     lambda: gen.weblike_t_device(1 << 14, seed=13, window=64)),
    ("web_wrap", lambda: gen.weblike_t(3000, seed=4, window=2000),
     lambda: gen.weblike_t_device(3000, seed=4, window=2000)),
    ("rmat", lambda: gen.rmat_t(12, 16 << 12, seed=11),
     lambda: gen.rmat_t_device(12, 16 << 12, seed=11)),
]


@pytest.mark.parametrize("name,host,device", SMALL, ids=[s[0] for s in SMALL])
def test_device_builders_match_host(name, host, device):
    hg, dg = host(), device()
    assert isinstance(dg, hb.DeviceCsrGraph)
    assert gen.graph_digest(hg) == gen.graph_digest(dg.to_host())


@pytest.mark.parametrize("name", ["config1", "config2", "config3", "config4"])
def test_device_builders_full_size_digest(name):
    """The device-built benchmark graphs are the graphs the reference ran on."""
    want = json.load(open(os.path.join(GOLDEN_DIR, "fullsize.json")))[name]["graph_digest"]
    g = gen.CONFIGS[name].build_device(torch.device("cuda", 0))
    assert g.n == json.load(open(os.path.join(GOLDEN_DIR, "fullsize.json")))[name]["n"]
    assert gen.graph_digest(g.to_host()) == want


def test_engine_on_device_transposed_graph():
    """The reference's pipeline (forward graph -> transpose -> engine) with the transpose
    on the device: registers identical to the golden run of the same graph."""
    case = next(c for c in golden_cases() if c["key"] == "random300_b6_s42_w5")
    off, suc = golden_graph(case)                  # the transpose the golden run used
    fwd = hb.transpose(hb.CsrGraph(off, suc))      # back to the forward graph (host)
    gT = hb.transpose_device(fwd)                  # and transposed again on the device
    st = hb.run(gT, hb.HyperBallConfig(params=hb.CounterParams(b=6, seed=42)))
    assert st.t == case["t"]
    assert (hashlib.sha256(st.register_matrix().tobytes()).hexdigest()
            == case["reg_digests"][-1])
