"""Probe: config 4's dense step with every successor id folded into a tiny hot set
(id mod K), i.e. the same instruction stream with every row load an L1/L2 hit.  The gap
to the real step is the memory latency the light kernel does not hide.

    python tools/latency_floor_probe.py K [bench args...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1308_2144_b200 import generators as gen  # noqa: E402
from paper_1308_2144_b200.graph import CsrGraph  # noqa: E402

K = int(sys.argv[1])
name = os.environ.get("PROBE_CONFIG", "config4")
orig = gen.BUILDERS[name]


def folded(th=None):
    g = orig(th)
    suc = (np.asarray(g.successors, dtype=np.int64) % K).astype(np.int32)
    return CsrGraph(np.asarray(g.offsets), suc)


gen.BUILDERS[name] = folded
import bench  # noqa: E402

sys.argv = ["bench.py", "--config", name] + sys.argv[2:]
bench.main()
