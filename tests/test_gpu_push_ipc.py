"""The fused push across two PROCESSES (tests/push_two_process.py): two ranks on one GPU,
each mapping the other's register buffers, change bitmaps and packed inboxes by CUDA IPC,
stepping with a gloo all-reduce as the barrier -- the cross-process path the simulated
ranks of test_gpu_distributed.py run sequentially in one process.  Both replicas must end
with the reference's registers."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import golden_cases, golden_graph

pytestmark = pytest.mark.gpu

CASES = {c["key"]: c for c in golden_cases()}
SCRIPT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "push_two_process.py")


@pytest.mark.parametrize("key,schedule,packed", [
    ("rmat12_b7_s42_w5", "degree", 1), ("rmat12_b7_s42_w5", "degree", 0),
    ("rmat12_b7_s42_w5", "identity", 1), ("disc14_b4_s42_w5", "degree", 1),
    ("web14_b8_s42_w5", "window", 1)])
def test_fused_push_two_processes(tmp_path, key, schedule, packed):
    pytest.importorskip("torch")
    case = CASES[key]
    off, suc = golden_graph(case)
    path = tmp_path / "g.npz"
    np.savez(path, off=off, suc=suc)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, SCRIPT, repo, str(port), str(path), str(case["b"]),
                          str(case["seed"]), schedule, str(packed)],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["t"] == case["t"]
    assert res["regs0"] == case["reg_digests"][-1]
    assert res["regs1"] == case["reg_digests"][-1]
