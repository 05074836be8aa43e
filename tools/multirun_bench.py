"""Time run_multi (R runs) batched vs one after the other on a device-built config.
usage: python tools/multirun_bench.py config5s 4"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1308_2144_b200 as hb  # noqa: E402
from paper_1308_2144_b200 import generators as gen  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config5s"
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfgd = gen.CONFIGS[name]
g = cfgd.build_device(torch.device("cuda", 0))
cfg = hb.HyperBallConfig(params=hb.CounterParams(b=cfgd.log2m, seed=cfgd.hash_seed))
for batch in (1, runs, 1, runs):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = hb.run_multi(g, cfg, runs, batch=batch)
    hs = [hb.finalize_harmonic(a) for _, a in out]
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    its = [s.t for s, _ in out]
    merged = sum(s._dev.merged_total for s, _ in out) if batch == 1 else None
    print(f"{name} runs={runs} batch={batch}: {dt:.3f} s  ({dt / runs * 1000:.1f} ms/run) "
          f"iterations {its}")
    del out, hs

# phase breakdown of one batched call
from paper_1308_2144_b200 import multirun as M  # noqa: E402
T = {"step": [], "init": 0.0}
orig_step, orig_init = M._Batch.step, M._Batch.__init__


def step(self, *a, **k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = orig_step(self, *a, **k)
    torch.cuda.synchronize()
    T["step"].append(round((time.perf_counter() - t0) * 1000, 2))
    return r


def init(self, *a, **k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    orig_init(self, *a, **k)
    torch.cuda.synchronize()
    T["init"] = round((time.perf_counter() - t0) * 1000, 2)


M._Batch.step, M._Batch.__init__ = step, init
torch.cuda.synchronize()
t0 = time.perf_counter()
out = hb.run_multi(g, cfg, runs, batch=runs)
torch.cuda.synchronize()
print("batched total ms", round((time.perf_counter() - t0) * 1000, 1), "init ms", T["init"],
      "steps ms", T["step"])
