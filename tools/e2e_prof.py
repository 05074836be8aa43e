import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1308_2144_b200 as hb
from paper_1308_2144_b200 import generators as gen, engine as E, schedule as S
g = gen.CONFIGS["config4"].build()
n, m = g.n, g.m
off_pin = torch.empty(n + 1, dtype=torch.int64, pin_memory=True); off_pin.numpy()[:] = g.offsets
suc_pin = torch.empty(m, dtype=torch.int32, pin_memory=True); suc_pin.numpy()[:] = g.successors
gp = hb.CsrGraph(off_pin.numpy(), suc_pin.numpy())
params = hb.CounterParams(b=8, seed=42)
for rep in range(2):
    torch.cuda.synchronize(); T = {}
    t0 = time.perf_counter()
    cfg = hb.HyperBallConfig(params=params, device=0)
    st = hb.initialize(gp, cfg); torch.cuda.synchronize(); T['init'] = time.perf_counter() - t0
    acc = hb.CentralityAccumulator(n)
    t1 = time.perf_counter()
    its = []
    while True:
        ti = time.perf_counter()
        nch = hb.iterate(gp, st, [acc])
        its.append(round((time.perf_counter() - ti) * 1000, 1))
        if nch == 0: break
    T['iters'] = time.perf_counter() - t1
    t2 = time.perf_counter(); fin = st.est; T['est_d2h'] = time.perf_counter() - t2
    t3 = time.perf_counter(); acc.on_converged(fin); T['on_conv'] = time.perf_counter() - t3
    t4 = time.perf_counter(); h = hb.finalize_harmonic(acc); c = hb.finalize_closeness(acc); l = hb.finalize_lin(acc); T['finalize'] = time.perf_counter() - t4
    print(rep, {k: round(v, 3) for k, v in T.items()}, its)
    del st, acc
# schedule-only timing
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    s = S.build_schedule(gp.offsets, gp.successors, 8, torch.device('cuda', 0))
    torch.cuda.synchronize(); print('schedule', time.perf_counter() - t)
    t = time.perf_counter(); x = torch.from_numpy(gp.successors).to('cuda', non_blocking=True); torch.cuda.synchronize(); print('succ h2d', time.perf_counter() - t, torch.from_numpy(gp.successors).is_pinned())
