import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1308_2144_b200 as hb
from paper_1308_2144_b200 import generators as gen
g = gen.CONFIGS["config3"].build()
params = hb.CounterParams(b=6, seed=42)
for rep in range(3):
    acc = hb.CentralityAccumulator(g.n)
    st = hb.run(g, hb.HyperBallConfig(params=params), [acc])
    b = acc._binding
    print("binding", b is not None, "stale", b.stale, "coreach_dev", b.coreach_dev is not None,
          "id match", b.coreach_host_id == id(acc.coreach))
    for which in ("harmonic", "closeness", "lin", "lin"):
        torch.cuda.synchronize(); t = time.perf_counter()
        out = b.finalize(which)
        print(which, round((time.perf_counter() - t) * 1000, 2), "ms")
    del st, acc, out, b
