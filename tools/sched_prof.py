"""Time the phases of initialize() (upload, schedule build, seed) for one config."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1308_2144_b200 as hb  # noqa: E402
from paper_1308_2144_b200 import generators as gen, schedule as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config5s"
ORDER = sys.argv[3] if len(sys.argv) > 3 else "auto"
cfgd = gen.CONFIGS[name]
g = cfgd.build()
n, m = g.n, g.m
off_pin = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
off_pin.numpy()[:] = g.offsets
suc_pin = torch.empty(m, dtype=torch.int32, pin_memory=True)
suc_pin.numpy()[:] = g.successors
dev = torch.device("cuda", 0)
orig = {k: getattr(S, k) for k in ("_as_device",)}
T = {}


def timed(label, fn):
    def w(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        T[label] = T.get(label, 0.0) + time.perf_counter() - t0
        return r
    return w


S._as_device = timed("upload", S._as_device)
L = hb._lib.hb()
for fn in ("hb_relabel_csr", "hb_sort_rows"):
    setattr(L, fn, timed(fn, getattr(L, fn)))
for rep in range(3):
    T.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = S.build_schedule(off_pin, suc_pin, cfgd.log2m, dev, ORDER)
    torch.cuda.synchronize()
    T["build_schedule_total"] = time.perf_counter() - t0
    print(rep, s.order, {k: round(v * 1000, 2) for k, v in T.items()})
    del s

if len(sys.argv) > 2 and sys.argv[2] == "torchprof":
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        s = S.build_schedule(off_pin, suc_pin, cfgd.log2m, dev, ORDER)
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
