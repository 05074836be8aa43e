"""Break down one end-to-end run (bench.py's e2e step) into phases.  The synchronize
after initialize() waits for the whole streamed upload, so "init" + iteration 1 here
overstate the pipelined run (bench.py's e2e has no sync there)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1308_2144_b200 as hb  # noqa: E402
from paper_1308_2144_b200 import generators as gen  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config4"
cfgd = gen.CONFIGS[name]
if name in gen.DEVICE_BUILDERS:      # R-MAT: built on the device, copied to the host
    g = cfgd.build_device(torch.device("cuda", 0)).to_host()
    torch.cuda.empty_cache()
else:
    g = cfgd.build()
n, m = g.n, g.m
off_pin = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
off_pin.numpy()[:] = g.offsets
suc_pin = torch.empty(m, dtype=torch.int32, pin_memory=True)
suc_pin.numpy()[:] = g.successors
gp = hb.CsrGraph(off_pin.numpy(), suc_pin.numpy())
params = hb.CounterParams(b=cfgd.log2m, seed=cfgd.hash_seed)
for rep in range(3):
    torch.cuda.synchronize()
    T = {}
    t0 = time.perf_counter()
    st = hb.initialize(gp, hb.HyperBallConfig(params=params, device=0,
                                              schedule=os.environ.get("HB_SCHEDULE", "auto")))
    torch.cuda.synchronize()
    T["init"] = time.perf_counter() - t0
    acc = hb.CentralityAccumulator(n)
    t1 = time.perf_counter()
    its = []
    while True:
        ti = time.perf_counter()
        nch = hb.iterate(gp, st, [acc])
        its.append((round((time.perf_counter() - ti) * 1000, 1), nch, st._dev.last_merged))
        if nch == 0:
            break
    T["iters"] = time.perf_counter() - t1
    t2 = time.perf_counter()
    fin = st.est
    fin.setflags(write=False)
    T["est_d2h"] = time.perf_counter() - t2
    t3 = time.perf_counter()
    acc.on_converged(fin)
    T["on_conv"] = time.perf_counter() - t3
    t4 = time.perf_counter()
    h = hb.finalize_harmonic(acc)
    t5 = time.perf_counter()
    c = hb.finalize_closeness(acc)
    t6 = time.perf_counter()
    lin = hb.finalize_lin(acc)
    T["finalize"] = time.perf_counter() - t4
    T["fin_h"], T["fin_c"], T["fin_l"] = t5 - t4, t6 - t5, time.perf_counter() - t6
    T["device_path"] = acc._binding is not None and not acc._binding.stale
    T["total"] = time.perf_counter() - t0
    print(rep, {k: round(v, 4) for k, v in T.items()})
    print("   iterations (ms, changed, merged arcs):", its)
    del st, acc, h, c, lin, fin
