"""HyperBall hot-path benchmark (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config config4]
    python bench.py --impl reference ...        # CPU reference arm (oracle port, all cores)

Metric (BASELINE.json): arcs x registers merged per second, and the union kernel's
fraction of the B200 HBM roofline.

* step   = one dense HyperBall iteration (iteration 1: every counter changed in the
           previous step, so every arc's source row is merged) over the whole synthetic
           graph, with the estimate and the fused harmonic/closeness/Lin accumulation --
           exactly one ``hb_union_step`` call plus the 16-byte changed-count read-back
           that ends every iteration.  Inputs are resident in HBM and larger than L2
           (config 4: 4.3 GB of registers), so no L2 flush is needed between steps.
* value  = m * 2^log2m / (device time per step), CUDA events on the launching stream,
           max over ranks.
* e2e    = the same metric through the public API a user calls: ``run(g, config,
           [CentralityAccumulator])`` + the three finalizers, from pinned host CSR arrays,
           with the host->device graph copy and the device->host result copy inside the
           timed region; arcs counted are the arcs actually merged over the whole run
           (source-skip aware, counted on the device).
* roofline = algorithmic bytes of one dense step, m*p (source rows) + 8(n+1) + 4m (CSR)
           + n*p (counter writes), over the union kernels' event
           time, against MEASURED_PEAKS.json hbm_gbs.
* cpu_baseline = the CPU oracle port (oracle/hb_oracle.c, pthreads over all host cores)
           doing the same dense step on a bounded sample of destination nodes.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

METRIC = "HyperBall arcs×registers merged/sec at 1/2/4/8 B200; % of HBM roofline"
UNIT = "arcs*registers/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peak():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out, _ = self.proc.communicate()
        return False

    def summary(self):
        sms, maxes, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sms.append(float(parts[0]))
                maxes.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sms:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sms), "sm_max_mhz": max(maxes),
                "reasons": sorted(reasons), "samples": len(sms)}


def build_graph(config_name: str):
    from paper_1308_2144_b200 import generators as gen
    t0 = time.perf_counter()
    g = gen.CONFIGS[config_name].build()
    log(f"[bench] built {config_name}: n={g.n} m={g.m} in {time.perf_counter() - t0:.1f}s")
    return g


def alg_bytes(n: int, m: int, p: int) -> int:
    """Algorithmic bytes of one dense step: source rows + CSR + counter writes."""
    return m * p + 8 * (n + 1) + 4 * m + n * p


# ------------------------------------------------------------------------ CPU arms

def cpu_dense_sample(g, b: int, seed: int, budget_s: float, threads: int, repeats: int = 1,
                     rotate: bool = False):
    """Time the oracle's dense union pass (hll_union_range restated, pthreads) on node
    ranges holding about `budget_s` seconds of work.  Returns a list of (arcs, seconds)."""
    import ctypes

    import oracle as orc
    L = orc.lib()
    n, p = g.n, 1 << b
    off = np.ascontiguousarray(g.offsets, np.int64)
    suc = np.ascontiguousarray(g.successors, np.int64)
    cur, est = orc.seed_registers(n, b, 5, seed)
    nxt = np.zeros_like(cur)
    nxt.fill(0)                                   # pre-fault
    chg_prev = np.ones(n, np.uint8)
    chg_now = np.zeros(n, np.uint8)
    new_est = np.zeros(n, np.float64)
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731

    def run_range(lo, hi):
        # arc-balanced sub-ranges over `threads` pthreads, like engine.py:351-390
        t0 = time.perf_counter()
        L.orc_iterate_range_mt(lo, hi, P(off), P(suc), P(cur), P(nxt), P(chg_prev),
                               P(chg_now), P(est), P(new_est), b, 1, threads)
        return int(off[hi] - off[lo]), time.perf_counter() - t0

    # calibrate on ~1/64 of the arcs
    hi0 = int(np.searchsorted(off, off[-1] // 64))
    a0, s0 = run_range(0, max(hi0, 1))
    rate = a0 / max(s0, 1e-6)
    want = max(int(rate * budget_s), 1)
    out = []
    lo = 0
    for _ in range(repeats):
        if int(off[-1]) - int(off[lo]) < want:      # not enough arcs left: wrap around
            lo = 0
        target = min(int(off[lo]) + want, int(off[-1]))
        hi = int(np.searchsorted(off, target))
        hi = max(min(hi, n), lo + 1)
        out.append(run_range(lo, hi))
        if rotate:
            lo = hi if hi < n else 0
    del cur, nxt
    return out, p


def _local_sub_csr_note():
    return ("contiguous destination-node ranges of the full graph, source rows read from the "
            "full register array")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1308_2144_b200 import generators as gen
    cfg = gen.CONFIGS[args.config]
    g = build_graph(args.config)
    threads = os.cpu_count() or 1
    per_step = max(0.5, min(20.0, args.ref_budget / max(args.steps + args.warmup, 1)))
    samples, p = cpu_dense_sample(g, cfg.log2m, cfg.hash_seed, per_step, threads,
                                  repeats=args.warmup + args.steps, rotate=True)
    timed = samples[args.warmup:]
    arcs = sum(a for a, _ in timed)
    secs = sum(s for _, s in timed)
    value = arcs * p / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * secs / len(timed), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": f"{args.config}: {cfg.description}", "n": g.n, "m": g.m,
                   "log2m": cfg.log2m, "hash_seed": cfg.hash_seed,
                   "step": "dense union pass (hll_union_range restated in C) over a "
                           "contiguous destination range of ~%.1f s of work" % per_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{len(timed)} dense-pass samples, {arcs} arcs total; "
                                   + _local_sub_csr_note()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------ GPU arm

def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_1308_2144_b200 as hb
    from paper_1308_2144_b200 import _lib
    from paper_1308_2144_b200 import generators as gen

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfgd = gen.CONFIGS[args.config]
    b, seed = cfgd.log2m, cfgd.hash_seed
    p = 1 << b
    t0 = time.perf_counter()
    g = cfgd.build_device(torch.device("cuda", local))     # GPU builder where one exists
    torch.cuda.synchronize()
    log(f"[bench] built {args.config} ({type(g).__name__}): n={g.n} m={g.m} in "
        f"{time.perf_counter() - t0:.1f}s")
    n, m = g.n, g.m
    host_graph = None

    def host_g():
        nonlocal host_graph
        if host_graph is None:
            host_graph = g.to_host() if hasattr(g, "to_host") else g
        return host_graph
    params = hb.CounterParams(b=b, seed=seed)

    # ---------------------------------------------------------------- device-resident step
    cfg = hb.HyperBallConfig(params=params, device=local, schedule=args.schedule)
    acc = hb.CentralityAccumulator(n)
    rs = comm = st = symm = None
    if world > 1:
        from paper_1308_2144_b200.distributed import CudaRankState, TorchComm
        comm = TorchComm()
        rs = CudaRankState(g, cfg, world, rank)
        sums = rs.bind_sums()
        dev = rs.dev
        symm = None
        if args.exchange == "push":
            from paper_1308_2144_b200.distributed import _ptr_array, setup_push
            symm = setup_push(rs)
    else:
        from paper_1308_2144_b200.engine import _bind_sums
        st = hb.initialize(g, cfg)
        dev = st._dev
        sums = _bind_sums(st, acc)
    s = dev.sched
    stream = dev.stream
    L = _lib.hb()
    # the config's outputs (BASELINE: config 5 is harmonic only): closeness and Lin need
    # sum_dist, harmonic needs sum_recip
    outputs = tuple(cfgd.outputs)
    need_dist = "closeness" in outputs or "lin" in outputs

    def step(ev0=None, ev1=None):
        """One dense iteration: union kernels (+ exchange of changed rows when N > 1: fused
        into the union epilogue with --exchange push, else pack / all-gather / scatter)."""
        npeer, pn, pc, clear = 0, None, None, 1
        if symm is not None:
            pnl, pcl = symm.peer_pointers(dev)
            npeer, pn, pc, clear = len(pnl), _ptr_array(pnl), _ptr_array(pcl), 0
        if ev0 is not None:
            ev0.record(stream)
        _lib.check(L.hb_union_step(
            n, s.light_lo, s.light_hi if dev.full_pass else s.light_hi_steady,
            s.offsets.data_ptr(), s.succ.data_ptr(),
            dev.cur.data_ptr(), dev.nxt.data_ptr(), dev.chg_prev.data_ptr(),
            dev.chg_now.data_ptr(), clear, dev.est.data_ptr(),
            sums.sum_dist.data_ptr() if need_dist else None,
            sums.sum_recip.data_ptr(), 1, dev.lc.data_ptr(), dev.alpha_p2, dev.lc_cut, b, 1,
            s.light_max_deg, s.heavy_nodes.data_ptr(), s.item_first.data_ptr(), s.n_heavy,
            s.finish_order.data_ptr(), s.n_mega, s.item_node.data_ptr(), s.item_beg.data_ptr(), s.n_items, s.item_arcs,
            s.partial.data_ptr(), dev.counts.data_ptr(), dev.counts.data_ptr() + 8,
            s.hot_rows, None, 0, 0, None, 0, None, npeer, pn, pc, stream.cuda_stream),
            "hb_union_step")
        if ev1 is not None:
            ev1.record(stream)
        nch, merged = (int(x) for x in dev.counts.cpu())   # the per-iteration termination read
        if symm is not None:
            # the all-reduce of the changed count is the barrier after which every peer's
            # pushed rows are visible; chg_prev stays all-ones so each step is iteration 1
            tot = torch.tensor([nch], dtype=torch.int64, device=dev.device)
            dist.all_reduce(tot)
        elif rs is not None:
            rs.refresh_unowned()
            ids, rows, k = rs.gather_changed()
            _, parts = comm.exchange(ids, rows, k)
            for ids_q, rows_q in parts:
                rs.apply_remote(ids_q, rows_q)
        return nch, merged

    launches_per_step = (s.light_hi > s.light_lo) + (s.n_items > 0) + (s.n_heavy > 0)
    if world > 1 and symm is None:
        launches_per_step += 2 + (world - 1)   # refresh, gather, one scatter per peer
    for _ in range(args.warmup):
        step()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    merged_check = None
    with ClockSampler(local) as clk:
        t_start.record(stream)
        for i in range(args.steps):
            nch, merged = step(*evs[i])
            merged_check = merged
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = t_start.elapsed_time(t_end)
    kernel_ms = [a.elapsed_time(b_) for a, b_ in evs]
    if world > 1:
        tt = torch.tensor([total_ms, sum(kernel_ms)], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms, ksum = tt.tolist()
    else:
        ksum = sum(kernel_ms)
    ms_per_step = total_ms / args.steps
    k_ms = ksum / args.steps
    if world > 1:
        mt = torch.tensor([merged_check], dtype=torch.int64, device="cuda")
        dist.all_reduce(mt)
        merged_check = int(mt.item())
    assert merged_check == m, (merged_check, m)   # dense step merges every arc
    value = m * p / (ms_per_step / 1000.0)
    peak, peak_src = measured_peak()
    B = alg_bytes(n, m, p)
    achieved = B / world / (k_ms / 1000.0) / 1e9    # per GPU: its share of B / its kernel time
    traffic = None
    tpath = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.config)
        except Exception:
            traffic = None
    clocks = clk.summary()

    # ---------------------------------------------------------------- whole run + e2e
    e2e = None
    whole = None
    if not args.no_e2e:
        # pinned host copies of the graph: the user-side buffers of the e2e call
        off_pin = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
        suc_pin = torch.empty(m, dtype=torch.int32, pin_memory=True)
        hg = host_g()
        off_pin.numpy()[:] = hg.offsets
        suc_pin.numpy()[:] = hg.successors
        gp = hb.CsrGraph(off_pin.numpy(), suc_pin.numpy())
        del st, rs, dev, sums, acc
        torch.cuda.empty_cache()
        runs = []
        for i in range(args.e2e_warmup + args.e2e_steps):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            acc2 = hb.CentralityAccumulator(n)
            cfg2 = hb.HyperBallConfig(params=params, device=local, schedule=args.schedule)
            if world > 1:
                from paper_1308_2144_b200.distributed import run_distributed
                st2 = run_distributed(gp, cfg2, [acc2], exchange=args.exchange)
            else:
                st2 = hb.run(gp, cfg2, [acc2])
            fins = [getattr(hb, f"finalize_{o}")(acc2) for o in outputs]
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            merged_total = (st2._dev.merged_total if world == 1 else st2.merged_total)
            iters = st2.t
            del st2, acc2, fins
            if i >= args.e2e_warmup:
                runs.append((dt, merged_total, iters))
        dt = max(r[0] for r in runs) if runs else float("nan")
        dts = [r[0] for r in runs]
        merged_total, iters = runs[-1][1], runs[-1][2]
        if world > 1:
            tt = torch.tensor([sum(dts)], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            sum_dt = tt.item()
        else:
            sum_dt = sum(dts)
        mean_dt = sum_dt / len(dts)
        e2e = {"value": merged_total * p / mean_dt, "unit": UNIT,
               "h2d_bytes_per_step": int(off_pin.numel() * 8 + suc_pin.numel() * 4),
               # the outputs and the 16-byte changed/merged counters read after every
               # iteration (the fused accumulator's final estimates stay on the device)
               "d2h_bytes_per_step": int(n * 8 * len(outputs) + 16 * iters),
               "seconds_per_run": mean_dt, "iterations": iters,
               "merged_arcs_per_run": merged_total,
               "what": "run(g, config, [CentralityAccumulator]) + finalize_{%s} from pinned "
                       "host CSR; graph upload, schedule, seed, all iterations to convergence "
                       "and result download timed" % ",".join(outputs)}
        whole = {"iterations": iters, "merged_arcs": merged_total,
                 "dense_equivalent_arcs": m * iters}

    # ---------------------------------------------------------------- CPU baseline
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        samples, _ = cpu_dense_sample(host_g(), b, seed, args.cpu_budget, threads, repeats=1)
        arcs, secs = samples[0]
        cpu = {"value": arcs * p / secs, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"one dense union pass (oracle/hb_oracle.c, {threads} pthreads) over "
                         f"destination nodes holding {arcs} of {m} arcs ({secs:.1f} s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic",
            "config": {"workload": f"{args.config}: {cfgd.description}", "n": n, "m": m,
                       "log2m": b, "register_width": 5, "hash_seed": seed,
                       "schedule": s.order, "heavy_nodes": s.n_heavy, "items": s.n_items,
                       "step": "one dense iteration (all sources changed): union + estimate + "
                               "fused accumulate for %s" % "/".join(outputs),
                       "l2": ("inputs larger than L2 (%.2f GB of registers + %.2f GB of CSR), "
                              "no flush" if n * p > 126e6 else
                              "registers (%.2f GB) + CSR (%.2f GB) partly L2-resident, no "
                              "flush: a small-graph line") % (n * p / 1e9,
                                                             (8 * (n + 1) + 4 * m) / 1e9),
                       "parallelism": (f"node-partition x{world}, {args.exchange} exchange"
                                       if world > 1 else "single GPU")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": B, "kernel_ms": k_ms,
                         "peak_source": peak_src,
                         "kernels": "hb_union_step (light%s)" % (
                             " + heavy items + finish" if s.n_items else "")},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "whole_run": whole,
            "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", default="config4")
    ap.add_argument("--schedule", default="auto", choices=["auto", "identity", "degree", "window"])
    ap.add_argument("--exchange", choices=["push", "allgather"], default="push",
                    help="N > 1: fused push over symmetric memory, or all-gather")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-warmup", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0,
                    help="seconds of CPU work in the cpu_baseline sample")
    ap.add_argument("--ref-budget", type=float, default=120.0,
                    help="total seconds of CPU work for --impl reference")
    args = ap.parse_args()
    if args.warmup < 3:
        log("[bench] warmup raised to 3 (timing rule)")
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
