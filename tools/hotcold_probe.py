"""Probe: dense-step time of config 5 restricted to arcs whose source is among the H
highest in-degree nodes ("hot") or outside them ("cold").  Tells how much of the step is
the random gather of rarely-read rows.

    python tools/hotcold_probe.py hot 4194304 [bench args...]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1308_2144_b200 import generators as gen  # noqa: E402
from paper_1308_2144_b200.graph import DeviceCsrGraph  # noqa: E402

which, H = sys.argv[1], int(sys.argv[2])
cfgname = os.environ.get("PROBE_CONFIG", "config5")
orig = gen.DEVICE_BUILDERS[cfgname]


def filtered(dev=None):
    g = orig(dev)
    off, suc = g.offsets, g.successors
    indeg = off[1:] - off[:-1]
    order = torch.argsort(-indeg, stable=True)
    rank = torch.empty_like(order)
    rank[order] = torch.arange(order.numel(), device=order.device)
    rank32 = rank.to(torch.int32)
    del rank, order, indeg
    m = suc.numel()
    mask = torch.empty(m, dtype=torch.bool, device=suc.device)
    step = 1 << 29
    for a in range(0, m, step):
        r = rank32[suc[a:a + step].long()]
        mask[a:a + step] = (r < H) if which == "hot" else (r >= H)
    cs = torch.zeros(m + 1, dtype=torch.int64, device=suc.device)
    torch.cumsum(mask, 0, out=cs[1:])
    new_off = cs[off]
    del cs
    new_suc = suc[mask]
    del mask, g, suc
    torch.cuda.empty_cache()
    print(f"[probe] {which} H={H}: m {m} -> {new_suc.numel()}", file=sys.stderr)
    return DeviceCsrGraph(new_off.contiguous(), new_suc.contiguous())


gen.DEVICE_BUILDERS[cfgname] = filtered
import bench  # noqa: E402

sys.argv = ["bench.py", "--config", cfgname] + sys.argv[3:]
bench.main()
