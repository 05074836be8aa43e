"""CPU-only tests: host logic, API validation, formats, and that the C-ABI library loads
and exports every symbol include/hyperball_b200.h declares (no compute without a GPU)."""

import ctypes
import hashlib
import io
import os
import re

import numpy as np
import pytest
import torch

import paper_1308_2144_b200 as hb
from paper_1308_2144_b200 import _lib, generators as gen
from paper_1308_2144_b200.hll import (CounterArray, CounterParams, alpha, estimator_constants,
                                      hash_items, lc_table, register_values)
from paper_1308_2144_b200.schedule import partition_bounds


def header_symbols():
    text = open(_lib.HEADER_PATH).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    L = ctypes.CDLL(_lib.HB_LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 10
    for name in syms:
        assert hasattr(L, name), name
    assert set(syms) == set(_lib.HB_SIGNATURES), "ctypes table out of sync with header"


def test_step_args_struct_layout():
    """ctypes' StepArgs and the library's hb_step_args agree (size and the struct_size
    check of hb_union_step_v2)."""
    L = _lib.hb()
    assert L.hb_step_args_size() == ctypes.sizeof(_lib.StepArgs)
    a = _lib.StepArgs(n=10, hi=10, t=1, b=4, nch_out=8)
    assert L.hb_union_step_v2(ctypes.byref(a)) == -1
    assert "null" in L.hb_last_error().decode()
    a.struct_size = 8
    assert L.hb_union_step_v2(ctypes.byref(a)) == -1
    assert "struct_size" in L.hb_last_error().decode()


def test_library_metadata_calls():
    L = _lib.hb()
    assert b"sm_100a" in L.hb_version()
    assert L.hb_min_log2m() == 4 and L.hb_max_log2m() >= 12
    assert L.hb_item_arcs(4) == 512 and L.hb_item_arcs(8) == 64
    # light/heavy threshold: 128 arcs for 16- / 32-register rows, 64 above
    assert L.hb_light_max_deg(4) == 128 and L.hb_light_max_deg(5) == 128
    assert L.hb_light_max_deg(6) == 64 and L.hb_light_max_deg(8) == 64
    assert L.hb_die_map_words(ctypes.c_void_p(4096 + 1000), 8192) == 1   # 5 chunks -> 1 word


def test_die_affine_items_are_opt_in(monkeypatch):
    from paper_1308_2144_b200.schedule import die_eligible
    monkeypatch.delenv("HB_DIE", raising=False)
    assert not die_eligible(1 << 28, 4, "degree")
    monkeypatch.setenv("HB_DIE", "1")
    assert die_eligible(1 << 28, 4, "degree")            # 4 GB of 16-byte rows
    assert not die_eligible(1 << 24, 4, "degree")        # 268 MB: below the 1 GB threshold
    assert not die_eligible(1 << 28, 4, "identity") and not die_eligible(1 << 28, 6, "degree")
    monkeypatch.setenv("HB_DIE_MIN_MB", "0")
    assert die_eligible(1 << 12, 5, "degree")


def _abi_args(name, **at):
    """Neutral arguments for C-ABI function `name` (NULL pointers, zeros, 1.0), with
    positional overrides at={index: value}."""
    out = []
    for k, ty in enumerate(_lib.HB_SIGNATURES[name][1]):
        v = None if ty is ctypes.c_void_p else (1.0 if ty is ctypes.c_double else 0)
        out.append(at.get(f"a{k}", v))
    return out


def test_c_abi_rejects_bad_arguments():
    """Argument validation happens before any CUDA call: error code -1 and a message
    (hb_last_error), on a host without a GPU too."""
    L = _lib.hb()

    def err(rc):
        assert rc == -1
        return L.hb_last_error().decode()
    # hb_union_step(n, lo, hi, ... t at 13, b at 17, nch_out at 30)
    base = dict(a0=10, a2=10, a13=1, a17=4, a30=ctypes.c_void_p(8))
    assert "null" in err(L.hb_union_step(*_abi_args("hb_union_step", **base)))
    assert "t" in err(L.hb_union_step(*_abi_args("hb_union_step", **{**base, "a13": 0})))
    assert "range" in err(L.hb_union_step(*_abi_args("hb_union_step", **{**base, "a2": 11})))
    assert "register_width" in err(L.hb_seed(*_abi_args("hb_seed", a2=5, a3=4, a4=9)))
    assert "hb_pack_registers" in err(L.hb_pack_registers(*_abi_args(
        "hb_pack_registers", a0=5, a1=2, a2=5)))
    assert "hb_unpack_registers" in err(L.hb_unpack_registers(*_abi_args(
        "hb_unpack_registers", a0=5, a1=4, a2=0)))
    assert "hb_sort_rows" in err(L.hb_sort_rows(*_abi_args("hb_sort_rows", a0=5, a2=1)))
    assert "hb_union_step_runs" in err(L.hb_union_step_runs(*_abi_args(
        "hb_union_step_runs", a0=10, a2=10, a14=1, a18=4, a19=5)))
    assert "hb_exact_seed" in err(L.hb_exact_seed(*_abi_args("hb_exact_seed", a0=100, a1=8)))
    assert "hb_estimate_rows" in err(L.hb_estimate_rows(*_abi_args(
        "hb_estimate_rows", a2=5, a3=4)))
    assert "hb_gather_changed" in err(L.hb_gather_changed(*_abi_args(
        "hb_gather_changed", a1=5, a4=4)))
    assert "hb_relabel_csr_rows" in err(L.hb_relabel_csr_rows(*_abi_args(
        "hb_relabel_csr_rows", a0=5, a1=3, a2=6)))
    assert "hb_mark_pull_filtered" in err(L.hb_mark_pull_filtered(*_abi_args(
        "hb_mark_pull_filtered", a0=5)))
    assert "hb_relabel_csr_src_rows" in err(L.hb_relabel_csr_src_rows(*_abi_args(
        "hb_relabel_csr_src_rows", a0=5, a1=3, a2=6)))
    assert "hb_sample_flagged_arcs" in err(L.hb_sample_flagged_arcs(*_abi_args(
        "hb_sample_flagged_arcs", a0=5, a3=8, a5=ctypes.c_void_p(8))))
    assert "hb_die_map" in err(L.hb_die_map(*_abi_args("hb_die_map", a1=1 << 20)))
    assert "hb_die_partition" in err(L.hb_die_partition(*_abi_args(
        "hb_die_partition", a0=5, a5=512, a6=4)))


def test_hash_and_register_pins(pins):
    p, _ = pins
    items = np.array([int(x) for x in p["hash_items"]["items"]], dtype=np.uint64)
    for key, vals in p["hash_items"]["values"].items():
        seed, replica = (int(x) for x in key.split(":"))
        got = hash_items(items, np.full(items.shape, replica, np.uint64), seed)
        assert [str(int(h)) for h in got] == vals
    hs = np.array([int(x) for x in p["register_values"]["hashes"]], dtype=np.uint64)
    for key, (idx, rho) in p["register_values"]["values"].items():
        b, w = (int(x) for x in key.split(":"))
        gi, gr = register_values(hs, CounterParams(b=b, register_width=w))
        assert gi.tolist() == idx and gr.tolist() == rho, key


def test_alpha_and_constants(pins):
    p, _ = pins
    for ps, a in p["alpha"].items():
        assert alpha(int(ps)) == a
    for ps, a2 in p["alpha_p2"].items():
        assert estimator_constants(int(ps))[0] == a2


def test_lc_table_matches_libm():
    import math
    for b in (4, 6, 8, 12):
        p = 1 << b
        t = lc_table(p)
        assert t[p] == 0.0 and t[p - 1] == float(p) * math.log(float(p) / (p - 1))


def test_hlla_blob_pins(pins):
    p, arrays = pins
    dense = arrays["hlla/dense"]
    for w, key in ((5, "hlla_blob_w5"), (6, "hlla_blob_w6")):
        blob = CounterArray.from_dense(dense, CounterParams(b=6, register_width=w, seed=9)).to_blob()
        assert hashlib.sha256(blob).hexdigest() == p[key]
        back = CounterArray.from_blob(blob)
        assert np.array_equal(back.to_dense(), dense)


@pytest.mark.parametrize("kw,exc", [(dict(b=3), ValueError), (dict(b=6, register_width=0), ValueError),
                                    (dict(b=6, register_width=9), ValueError)])
def test_counter_params_validation(kw, exc):
    with pytest.raises(exc):
        CounterParams(**kw)


def test_config_validation():
    with pytest.raises(ValueError):
        hb.HyperBallConfig(backend="nope")
    with pytest.raises(ValueError):
        hb.HyperBallConfig(workers=0)
    with pytest.raises(ValueError):
        hb.HyperBallConfig(schedule="random")
    assert hb.HyperBallConfig(backend="hll").backend == "probabilistic"


def test_engine_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    g = hb.CsrGraph([0, 1, 1], [1])
    with pytest.raises(RuntimeError, match="CUDA"):
        hb.run(g, hb.HyperBallConfig(params=CounterParams(b=4)))


def test_exact_backend_config():
    """backend="exact" is accepted (and still needs the device: no CPU fallback);
    unknown backends are rejected (engine.py:82-97)."""
    assert hb.HyperBallConfig(backend="exact").backend == "exact"
    assert hb.HyperBallConfig(backend="cuda").backend == "probabilistic"
    assert hb.HyperBallConfig(backend="hll").backend == "probabilistic"
    with pytest.raises(ValueError):
        hb.HyperBallConfig(backend="bitmap")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    g = hb.CsrGraph([0, 1, 1], [1])
    with pytest.raises(RuntimeError, match="CUDA"):
        hb.initialize(g, hb.HyperBallConfig(backend="exact"))


def test_graph_roundtrip_and_transpose():
    rng = np.random.default_rng(1)
    s, d = rng.integers(0, 50, 300), rng.integers(0, 50, 300)
    g = hb.CsrGraph.from_edges(s, d, n=50)
    assert all((np.diff(g.successors_of(v)) > 0).all() for v in range(50))
    gt = hb.transpose(g)
    assert hb.transpose(gt) == g
    buf = io.BytesIO()
    hb.write_binary(g, buf)
    assert len(buf.getvalue()) == 20 + 8 * 51 + 8 * g.m
    buf.seek(0)
    assert hb.read_binary(buf) == g


def test_generator_matches_reference_normalisation():
    """G^T from the C builder equals transpose(from_edges(arcs)) minus self-loops."""
    rng = np.random.default_rng(2)
    n = 300
    s = rng.integers(0, n, 3000).astype(np.uint32)
    d = rng.integers(0, n, 3000).astype(np.uint32)
    gt = gen.from_arcs_t(n, s, d, threads=3)
    keep = s != d
    want = hb.transpose(hb.CsrGraph.from_edges(s[keep], d[keep], n=n))
    assert gt == want


def test_generator_deterministic_across_threads():
    a = gen.rmat_t(11, 8 << 11, seed=5, threads=1)
    b = gen.rmat_t(11, 8 << 11, seed=5, threads=7)
    assert gen.graph_digest(a) == gen.graph_digest(b)


@pytest.mark.parametrize("n,w", [(10, 4), (7, 8), (1000, 3), (0, 2)])
def test_partition_bounds_cover(n, w):
    b = partition_bounds(n, w)
    assert b[0] == 0 and b[-1] == n and all(b[i] <= b[i + 1] for i in range(w))
    # round-robin deal sizes
    assert [b[r + 1] - b[r] for r in range(w)] == [len(range(r, n, w)) for r in range(w)]


def test_discount_spec_mirrors_reference_validation():
    from paper_1308_2144_b200 import DiscountSpec
    with pytest.raises(ValueError):
        DiscountSpec("nope")
    with pytest.raises(ValueError):
        DiscountSpec.from_table([1.0, 2.0], 0.5)          # increasing
    with pytest.raises(ValueError):
        DiscountSpec(kind="table", table=(1.0,))          # no tail
    assert DiscountSpec.preset("log").name == "log" and DiscountSpec.preset("log").kind == "logarithmic"
    t = DiscountSpec.from_table([1.0, 0.5], 0.25)
    assert [t.value(k) for k in (1, 2, 3, 9)] == [1.0, 0.5, 0.25, 0.25]
    assert DiscountSpec.preset("harmonic").device_factor(4) == (True, 0.0)
    assert DiscountSpec.preset("quad").device_factor(4) == (False, 1.0 / 16.0)


def test_multi_run_aggregate_semantics():
    runs = [np.array([1.0, 2.0, 4.0]), np.array([3.0, 2.0, 0.0])]
    mean, std = hb.multi_run_aggregate(runs)
    assert mean.tolist() == [2.0, 2.0, 2.0]
    assert np.allclose(std, np.vstack(runs).std(axis=0, ddof=1))
    m1, s1 = hb.multi_run_aggregate(runs[:1])
    assert s1 is None and m1.tolist() == [1.0, 2.0, 4.0]
    with pytest.raises(ValueError):
        hb.multi_run_aggregate([])
    with pytest.raises(ValueError):
        hb.multi_run_aggregate([np.zeros(2), np.zeros(3)])


@pytest.mark.parametrize("nslices,align", [(8, 64), (3, 16), (16, 1)])
def test_upload_slice_rows(nslices, align):
    """Streamed-upload slices: cover [0, n], strictly increasing, inner bounds aligned to
    the chunk window, arcs roughly balanced."""
    from paper_1308_2144_b200.schedule import slice_rows
    rng = np.random.default_rng(nslices)
    deg = rng.zipf(2.1, 100_000).clip(max=10_000)
    off = np.zeros(deg.size + 1, np.int64)
    np.cumsum(deg, out=off[1:])
    rows = slice_rows(off, nslices, align)
    assert rows[0] == 0 and rows[-1] == deg.size and np.all(np.diff(rows) > 0)
    assert np.all(rows[1:-1] % align == 0) and len(rows) <= nslices + 1
    arcs = np.diff(off[rows])
    assert arcs.max() <= off[-1] / nslices + deg.max() + align * deg.max()


def test_bench_reference_arm_json(tmp_path):
    """bench.py --impl reference (the CPU arm the driver runs) prints one JSON line with
    the contract's keys; a non-zero rank prints nothing."""
    import json
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, os.path.join(repo, "bench.py"), "--impl", "reference", "--config",
           "config1", "--steps", "2", "--warmup", "3", "--ref-budget", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, check=True).stdout
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    # no product library in the reference arm; its config dict is the one the B200 arm
    # prints for the same workload
    assert d["mapped_repo_libs"] == ["oracle/liborc.so"], d["mapped_repo_libs"]
    sys.path.insert(0, repo)
    import bench
    g = gen.BUILDERS["config1"]()
    assert d["config"] == bench.bench_config(gen.CONFIGS["config1"], g.n, g.m)
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0 and not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]


def test_sm100a_sass_uses_tma_gather_and_3input_max():
    """The built library is sm_100a code using the Blackwell features the design relies
    on: TMA tile::gather4 for the p = 256 row gathers (with mbarrier completion) and the
    3-input 16x2 integer max for the byte-wise union."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "-sass", _lib.HB_LIB_PATH], capture_output=True, text=True,
                         timeout=300).stdout
    assert "sm_100a" in out or "SM100" in out.upper()
    for op in ("UTMALDG.2D.GATHER4", "SYNCS.PHASECHK.TRANS64", "VIMNMX3.U16x2"):
        assert op in out, op


def test_oracle_carries_identical_graph_builders():
    """bench.py's reference arm builds its graph with the oracle library's copy of the
    builders (no product .so in that process): same bytes as libhbgraph.so."""
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, os; sys.path.insert(0, %r)\n"
        "from paper_1308_2144_b200 import _lib\n"
        "_lib.use_graph_library(os.path.join(%r, 'oracle', 'liborc.so'))\n"
        "from paper_1308_2144_b200 import generators as gen\n"
        "print(gen.graph_digest(gen.BUILDERS['config1']()))\n"
        "print(gen.graph_digest(gen.weblike_t(1 << 14, seed=3)))\n"
        "print(gen.graph_digest(gen.disconnected_t(1 << 14, 1 << 13, 0.1, 6.0, seed=2)))\n"
        "print(open('/proc/self/maps').read().count('libhbgraph'))\n"
    ) % (repo, repo)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         check=True).stdout.split()
    assert out[3] == "0"
    assert out[0] == gen.graph_digest(gen.BUILDERS["config1"]())
    assert out[1] == gen.graph_digest(gen.weblike_t(1 << 14, seed=3))
    assert out[2] == gen.graph_digest(gen.disconnected_t(1 << 14, 1 << 13, 0.1, 6.0, seed=2))


def _tgold():
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                             "transpose.npz"))
    return z, [str(x) for x in z["names"]]


def test_transpose_matches_reference_fixtures():
    """graph.transpose (host) == the reference's transpose (graph.py:145-155) on forward
    graphs with duplicate arcs, self-loops and empty rows (tests/golden/transpose.npz)."""
    z, names = _tgold()
    for nm in names:
        g = hb.CsrGraph(z[f"{nm}/offsets"], z[f"{nm}/successors"])
        t = hb.transpose(g)
        assert np.array_equal(np.asarray(t.offsets, np.int64), z[f"{nm}/t_offsets"]), nm
        assert np.array_equal(np.asarray(t.successors, np.int64), z[f"{nm}/t_successors"]), nm


def test_arc_list_builder_matches_reference_from_edges():
    """generators.from_arcs_t (graphgen.c: transpose + normalise an arc list, self-loops
    dropped) == the reference's transpose(from_edges(...)) of the self-loop-free arcs."""
    z, names = _tgold()
    for nm in names:
        if f"{nm}/arcs_src" not in z:
            continue
        src, dst = z[f"{nm}/arcs_src"], z[f"{nm}/arcs_dst"]
        n = int(z[f"{nm}/from_edges_offsets"].size - 1)
        g = gen.from_arcs_t(n, src, dst)
        assert np.array_equal(np.asarray(g.offsets, np.int64), z[f"{nm}/noloop_t_offsets"]), nm
        assert np.array_equal(np.asarray(g.successors, np.int64),
                              z[f"{nm}/noloop_t_successors"]), nm
