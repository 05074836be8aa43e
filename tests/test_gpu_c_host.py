"""The C-ABI from a non-Python host: tests/c_host/hb_host.c (plain C, gcc, linked against
libhyperball_b200.so and the CUDA runtime) seeds, steps with hb_union_step_v2 until no
counter changes and finalizes; its registers, iteration count and centralities must be
the golden ones produced by running the reference."""

import hashlib
import os
import subprocess

import numpy as np
import pytest

from conftest import golden, golden_cases, golden_graph

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = {c["key"]: c for c in golden_cases()}


@pytest.fixture(scope="module")
def host_bin(tmp_path_factory):
    out = tmp_path_factory.mktemp("chost") / "hb_host"
    lib = os.path.join(REPO, "paper_1308_2144_b200")
    cmd = ["gcc", "-O2", "-std=c11", "-o", str(out), os.path.join(REPO, "tests", "c_host", "hb_host.c"),
           "-I", os.path.join(REPO, "include"), "-I", "/usr/local/cuda/include",
           "-L", lib, "-lhyperball_b200", "-L", "/usr/local/cuda/lib64", "-lcudart", "-lm",
           f"-Wl,-rpath,{lib}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return str(out)


@pytest.mark.parametrize("key", ["random300_b6_s42_w5", "rmat12_b7_s42_w5", "web14_b8_s42_w5",
                                 "disc14_b4_s42_w5", "config1_b6_s42_w5"])
def test_c_host_matches_reference(host_bin, tmp_path, key):
    case = CASES[key]
    off, suc = golden_graph(case)
    n, m = off.shape[0] - 1, int(off[-1])
    gpath, opath = tmp_path / "g.bin", tmp_path / "o.bin"
    with open(gpath, "wb") as f:
        f.write(np.array([n, m], np.int64).tobytes())
        f.write(np.ascontiguousarray(off, np.int64).tobytes())
        f.write(np.ascontiguousarray(suc, np.int32).tobytes())
    r = subprocess.run([host_bin, str(gpath), str(case["b"]), str(case["seed"]), str(opath)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    raw = opath.read_bytes()
    p = 1 << case["b"]
    t = int(np.frombuffer(raw[:8], np.int64)[0])
    regs = np.frombuffer(raw[8:8 + n * p], np.uint8).reshape(n, p)
    rest = np.frombuffer(raw[8 + n * p:], np.float64)
    h, c, lin = rest[:n], rest[n:2 * n], rest[2 * n:]
    assert t == case["t"]
    assert hashlib.sha256(regs.tobytes()).hexdigest() == case["reg_digests"][-1]
    _, arrays = golden()
    for name, got in (("harmonic", h), ("closeness", c), ("lin", lin)):
        assert np.array_equal(got.view(np.uint64), arrays[f"{key}/{name}"].view(np.uint64)), name
