"""Two ranks in two processes running the fused push for real (tests/test_gpu_push_ipc.py).

Both processes use cuda:0 (the pool hands out one GPU): each rank allocates its own
register double buffer, change bitmaps and (packed) inboxes, the other rank maps them by
CUDA IPC (torch.multiprocessing), and the union epilogue of each rank stores into the
other's buffers exactly as over NVLink between two GPUs.  The barrier is a gloo
all-reduce of the changed counts after each rank has synchronised its stream (the
kernels end with a system-scope fence).  No kernel waits on the other rank's kernels --
the push is fire-and-forget -- so time-slicing one GPU between the processes cannot
deadlock.

usage: python tests/push_two_process.py <repo> <port> <graph.npz> <b> <seed> <schedule>
       <packed 0/1>   -> prints one JSON line (t, register and estimate digests) per rank 0
"""

import hashlib
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def worker(rank, argv, q_out, q_in, res_q):
    repo, port, path, b, seed, schedule, packed = argv
    sys.path.insert(0, repo)
    import paper_1308_2144_b200 as hb
    from paper_1308_2144_b200 import distributed as D
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=2)
    d = np.load(path)
    g = hb.CsrGraph(d["off"], d["suc"])
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=int(b), seed=int(seed)),
                             schedule=schedule)
    st = D.CudaRankState(g, cfg, 2, rank)
    dev = st.dev
    n, p = dev.n, dev.p
    pstride = D.packed_push_stride(st, bool(int(packed)))
    # this rank's buffers (what SymmetricBuffers puts in symmetric memory)
    regs = torch.empty((2, n, p), dtype=torch.uint8, device=dev.device)
    bits = torch.empty((2, dev.chg_prev.numel()), dtype=torch.int32, device=dev.device)
    regs[0].copy_(dev.cur)
    regs[1].copy_(dev.nxt)
    bits[0].copy_(dev.chg_prev)
    bits[1].zero_()
    dev.cur, dev.nxt = regs[0], regs[1]
    dev.chg_prev, dev.chg_now = bits[0], bits[1]
    inbox = (torch.zeros((2, n, pstride), dtype=torch.uint8, device=dev.device)
             if pstride else None)
    prev_copy = torch.zeros_like(dev.chg_prev) if pstride else None
    torch.cuda.synchronize()
    # exchange the buffers by CUDA IPC: the peer's tensors map the same device memory
    q_out.put((regs, bits, inbox))
    p_regs, p_bits, p_inbox = q_in.get()
    dist.barrier()
    t = 0
    while True:
        t += 1
        # peer addresses: its nxt (or its step-t inbox) and its chg_now, in this step's
        # buffer parity (both ranks swap in lockstep)
        k_nxt = 1 if (t % 2 == 1) else 0
        if pstride:
            rows = p_inbox[t & 1].data_ptr()
        else:
            rows = p_regs[k_nxt].data_ptr()
        chg = p_bits[k_nxt].data_ptr()
        nch = D.push_step(st, t, t == 1, [rows], [chg], pstride, prev_copy)
        torch.cuda.synchronize()                     # our stores are done (+ fenced)
        tot = torch.tensor([nch], dtype=torch.int64)
        dist.all_reduce(tot)                         # the barrier of the step
        if pstride:
            D.unpack_inbox(st, inbox[t & 1], prev_copy)
        st.swap()
        torch.cuda.synchronize()
        if int(tot.item()) == 0:
            break
    regs_h = dev.to_host(dev.cur)
    est_h = dev.est.cpu()
    dist.barrier()
    res_q.put((rank, t, regs_h, est_h.numpy(), st.lo, st.hi))
    dist.barrier()
    dist.destroy_process_group()


def main():
    argv = sys.argv[1:8]
    ctx = mp.get_context("spawn")
    q01, q10, res_q = ctx.Queue(), ctx.Queue(), ctx.Queue()
    procs = [ctx.Process(target=worker, args=(0, argv, q01, q10, res_q)),
             ctx.Process(target=worker, args=(1, argv, q10, q01, res_q))]
    for pr in procs:
        pr.start()
    got = {}
    for _ in range(2):
        r, t, regs, est, lo, hi = res_q.get(timeout=600)
        got[r] = (t, regs, est, lo, hi)
    for pr in procs:
        pr.join(timeout=120)
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    (t0, r0, e0, lo0, hi0), (t1, r1, e1, lo1, hi1) = got[0], got[1]
    assert t0 == t1
    # estimates are per owned range (internal order); registers are full replicas
    print(json.dumps({"t": t0,
                      "regs0": hashlib.sha256(np.ascontiguousarray(r0).tobytes()).hexdigest(),
                      "regs1": hashlib.sha256(np.ascontiguousarray(r1).tobytes()).hexdigest()}))


if __name__ == "__main__":
    main()
