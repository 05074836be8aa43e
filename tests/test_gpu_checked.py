"""The bounds-checked build (HB_CHECKED, libhyperball_b200_checked.so): every indexed
access of the union kernels is asserted on the device (successor ids, CSR positions, row
indices, shared-memory slots, TMA rows, work items).  compute-sanitizer is closed on the
GPU pool, so this is the out-of-bounds evidence: the whole sanitizer workload
(tools/sanitize_workload.py -- TMA p = 256, heavy items, frontier marking, fused push
and all-gather on simulated ranks, batched runs, exact backend, checkpoints, device
builders) runs clean under it, and a deliberately corrupt graph is caught."""

import os
import subprocess
import sys

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu

CHECKED = os.path.join(REPO, "paper_1308_2144_b200", "libhyperball_b200_checked.so")


def _run(args, timeout=900):
    if not os.path.exists(CHECKED):
        pytest.skip("checked build missing (make -C paper_1308_2144_b200/csrc checked)")
    env = dict(os.environ, HB_LIB=CHECKED)
    return subprocess.run([sys.executable] + args, capture_output=True, text=True,
                          timeout=timeout, env=env, cwd=REPO)


def test_sanitize_workload_clean_under_checked_build():
    r = _run([os.path.join(REPO, "tools", "sanitize_workload.py")])
    progress = [ln for ln in r.stdout.splitlines() if "HB_CHECKED" not in ln]
    violations = [ln for ln in r.stdout.splitlines() if "HB_CHECKED" in ln]
    assert r.returncode == 0, "\n".join(progress[-20:] + violations[:5]) + r.stderr[-2000:]
    assert "sanitize workload ok" in r.stdout
    assert "HB_CHECKED violation" not in r.stdout + r.stderr


def test_checked_build_catches_an_out_of_range_id():
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import numpy as np, torch, paper_1308_2144_b200 as hb\n"
        "from paper_1308_2144_b200 import _lib\n"
        "assert _lib.HB_LIB_PATH.endswith('_checked.so')\n"
        "off = torch.tensor([0, 2, 3, 3, 4], dtype=torch.int64).cuda()\n"
        "suc = torch.tensor([1, 2, 0, 4], dtype=torch.int32).cuda()   # id 4 == n\n"
        "hb.run(hb.DeviceCsrGraph(off, suc),\n"
        "       hb.HyperBallConfig(params=hb.CounterParams(b=6, seed=1), schedule='identity'))\n"
        "torch.cuda.synchronize()\n"
        "print('NOT CAUGHT')\n" % REPO)
    r = _run(["-c", code], timeout=300)
    out = r.stdout + r.stderr
    assert "NOT CAUGHT" not in out
    assert "HB_CHECKED violation" in out, out[-3000:]
