"""Multi-rank protocol of paper_1308_2144_b200.distributed on CPU: world size 2 over gloo.

The driver (partition, refresh of remote rows, changed-row all-gather whose counts give
the global termination count, scatter) is the production code; the per-rank compute is
the CPU oracle (test infrastructure), since this container has no GPU.  Results must be
bit-identical to the reference's golden outputs.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as orc
from conftest import golden, golden_cases, golden_graph
from paper_1308_2144_b200 import CentralityAccumulator, CounterParams, CsrGraph, HyperBallConfig
from paper_1308_2144_b200.distributed import run_distributed
from paper_1308_2144_b200.schedule import partition_bounds


class OracleRankState:
    """CPU twin of CudaRankState (identity order, oracle compute, numpy arrays)."""

    def __init__(self, off, suc, b, seed, world, rank):
        self.off = np.ascontiguousarray(off, np.int64)
        self.suc = np.ascontiguousarray(suc, np.int64)
        self.n = self.off.shape[0] - 1
        self.b, self.p = b, 1 << b
        bounds = partition_bounds(self.n, world)
        self.lo, self.hi = bounds[rank], bounds[rank + 1]
        self.cur, self.est = orc.seed_registers(self.n, b, 5, seed)
        self.nxt = np.zeros_like(self.cur)
        self.chg_prev = np.ones(self.n, np.uint8)
        self.chg_now = np.zeros(self.n, np.uint8)
        self.sum_dist = np.zeros(self.n)
        self.sum_recip = np.zeros(self.n)
        self.sums = None

    def bind_sums(self, specs=()):
        assert not specs, "the CPU twin folds no discounts"
        self.sums = True

    def local_step(self, t, dense):
        import ctypes
        P = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        self.chg_now[:] = 0
        new_est = self.est.copy()
        nch = orc.lib().orc_union_range(self.lo, self.hi, P(self.off), P(self.suc), P(self.cur),
                                        P(self.nxt), P(self.chg_prev), P(self.chg_now),
                                        P(self.est), P(new_est), self.b, 1)
        lo, hi = self.lo, self.hi
        if hi > lo:
            sd, sr = self.sum_dist[lo:hi].copy(), self.sum_recip[lo:hi].copy()
            old, new = self.est[lo:hi].copy(), new_est[lo:hi].copy()
            orc.lib().orc_accumulate(hi - lo, t, P(old), P(new), P(sd), P(sr))
            self.sum_dist[lo:hi], self.sum_recip[lo:hi] = sd, sr
            self.est[lo:hi] = new
        return int(nch)

    def refresh_unowned(self):
        mask = self.chg_prev.astype(bool).copy()
        mask[self.lo:self.hi] = False
        self.nxt[mask] = self.cur[mask]

    def gather_changed(self):
        ids = np.flatnonzero(self.chg_now[self.lo:self.hi]) + self.lo
        rows = self.nxt[ids]
        return (torch.from_numpy(ids.astype(np.int32)), torch.from_numpy(rows.copy()),
                int(ids.size))

    def apply_remote(self, ids, rows):
        i = ids.numpy().astype(np.int64)
        self.nxt[i] = rows.numpy()
        self.chg_now[i] = 1

    def swap(self):
        self.cur, self.nxt = self.nxt, self.cur
        self.chg_prev, self.chg_now = self.chg_now, self.chg_prev

    def per_node(self):
        return {"est": torch.from_numpy(self.est), "sum_dist": torch.from_numpy(self.sum_dist),
                "sum_recip": torch.from_numpy(self.sum_recip)}

    def to_original(self, x):
        return x.numpy().copy()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, key, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        case = next(c for c in golden_cases() if c["key"] == key)
        off, suc = golden_graph(case)
        b, seed = case["b"], int(case["seed"])
        g = CsrGraph(off, suc)
        acc = CentralityAccumulator(g.n)
        cfg = HyperBallConfig(params=CounterParams(b=b, seed=seed))
        res = run_distributed(g, cfg, [acc], state_factory=lambda: OracleRankState(
            off, suc, b, seed, world, rank))
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), t=res.t, est=res.est,
                 sum_dist=acc.sum_dist, sum_recip=acc.sum_recip, coreach=acc.coreach)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("key,world", [("random300_b6_s42_w5", 2), ("disc14_b4_s42_w5", 2),
                                       ("dag300_b4_s42_w5", 3), ("isolated5_b6_s42_w5", 2)])
def test_gloo_world_matches_reference(key, world, tmp_path):
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, key, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    case = next(c for c in golden_cases() if c["key"] == key)
    _, arrays = golden()
    for r in range(world):
        got = np.load(tmp_path / f"r{r}.npz")
        assert int(got["t"]) == case["t"]
        for name in ("sum_dist", "sum_recip", "coreach"):
            want = arrays[f"{key}/{name}"]
            assert np.array_equal(got[name].view(np.uint64), want.view(np.uint64)), (r, name)
