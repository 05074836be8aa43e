"""Compute side of the multi-GPU step on ONE GPU: rank 0 of a world of W builds its
rank-local schedule (degree deal, owned rows only) and runs its dense union step with no
peers -- the per-rank kernel time a W-GPU run would overlap with the exchange (DESIGN.md
section 6's model; not a multi-GPU measurement).
usage: python tools/rank_step_bench.py [config] [worlds, e.g. 1,2,4,8] [exchange-like pushes: 0]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1308_2144_b200 as hb  # noqa: E402
from paper_1308_2144_b200 import generators as gen  # noqa: E402
from paper_1308_2144_b200.distributed import CudaRankState  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config5s"
worlds = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8").split(",")]
cfgd = gen.CONFIGS[name]
dev = torch.device("cuda", 0)
g = cfgd.build_device(dev) if name in gen.DEVICE_BUILDERS else cfgd.build()
params = hb.CounterParams(b=cfgd.log2m, seed=cfgd.hash_seed)
for w in worlds:
    for rank in sorted({0, w - 1}):
        cfg = hb.HyperBallConfig(params=params, device=0, schedule=os.environ.get("HB_SCHEDULE", "auto"))
        st = CudaRankState(g, cfg, world=w, rank=rank)
        st.bind_sums()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for it in range(6):
            st.dev.prev_all = True
            st.dev.chg_prev.fill_(-1)                 # every source changed: iteration 1 again
            ev0.record()
            nch = st.local_step(1, True)
            ev1.record()
            torch.cuda.synchronize()
            if it >= 2:
                ms.append(ev0.elapsed_time(ev1))
        s = st.dev.sched
        print(f"{name} W={w} rank={rank}: rows [{st.lo}, {st.hi}) arcs {s.m} items {s.n_items} "
              f"dense step {sum(ms) / len(ms):.3f} ms (changed {nch})", flush=True)
        del st
        torch.cuda.empty_cache()
