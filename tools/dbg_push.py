import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle')
import paper_1308_2144_b200 as hb
from paper_1308_2144_b200 import distributed as D
from conftest import golden_cases, golden_graph
case = {c["key"]: c for c in golden_cases()}["disc14_b4_s42_w5"]
off, suc = golden_graph(case)
g = hb.CsrGraph(off, suc)
cfg = hb.HyperBallConfig(params=hb.CounterParams(b=4, seed=42), schedule="degree")
def run(packed, T):
    states = [D.CudaRankState(g, cfg, 2, r) for r in range(2)]
    ps = D.packed_push_stride(states[0], packed)
    inb = {id(s): torch.zeros((2, s.n, max(ps,1)), dtype=torch.uint8, device=s.dev.device) for s in states}
    pc = {id(s): torch.zeros_like(s.dev.chg_prev) for s in states}
    hist = []
    for t in range(T):
        dense = t == 0
        for s in states:
            peers = [q for q in states if q is not s]
            rows = [inb[id(q)][(t+1)&1].data_ptr() for q in peers] if ps else [q.dev.nxt.data_ptr() for q in peers]
            D.push_step(s, t+1, dense, rows, [q.dev.chg_now.data_ptr() for q in peers], ps, pc[id(s)])
        if ps:
            for s in states: D.unpack_inbox(s, inb[id(s)][(t+1)&1], pc[id(s)])
        for s in states: s.swap()
        torch.cuda.synchronize()
        hist.append([ (s.dev.cur.cpu().numpy().copy(), s.dev.chg_prev.cpu().numpy().copy()) for s in states])
    return states, hist
T = 10
sa, ha = run(False, T)
sb, hb_ = run(True, T)
print("lo/hi", [(s.lo, s.hi) for s in sa], "light", [(s.dev.sched.light_lo, s.dev.sched.light_hi, s.dev.sched.light_hi_steady) for s in sa])
for t in range(T):
    for r in range(2):
        ra, ca = ha[t][r]; rb, cb = hb_[t][r]
        bad = np.nonzero((ra != rb).any(1))[0]
        cbad = np.nonzero(ca != cb)[0]
        if len(bad) or len(cbad):
            print("iter", t+1, "rank", r, "bad rows", len(bad), bad[:10], "bad chg words", len(cbad))
            if len(bad):
                v = bad[0]; print("  row a", ra[v], "\n  row b", rb[v])
    if any(len(np.nonzero((ha[t][r][0] != hb_[t][r][0]).any(1))[0]) for r in range(2)): break
