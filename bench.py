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


def mapped_repo_libs():
    """In-tree shared libraries mapped by this process (evidence of which native code ran:
    the reference arm maps only oracle/liborc.so, the B200 arm the kernel library)."""
    try:
        with open("/proc/self/maps") as fh:
            paths = {ln.split()[-1] for ln in fh if ln.rstrip().endswith(".so")}
    except OSError:
        return None
    root = os.path.realpath(REPO)
    return sorted(os.path.relpath(p_, root) for p_ in paths
                  if os.path.realpath(p_).startswith(root + os.sep))


def alg_bytes(n: int, m: int, p: int) -> int:
    """Algorithmic bytes of one dense step: source rows + CSR + counter writes."""
    return m * p + 8 * (n + 1) + 4 * m + n * p


# ------------------------------------------------------------------------ CPU arms

def cpu_dense_sample(g, b: int, seed: int, budget_s: float, threads: int, repeats: int = 1,
                     rotate: bool = False):
    """Time the oracle's dense step on node ranges holding about `budget_s` seconds of
    work: the union pass (hll_union_range restated, arc-balanced pthread ranges as
    engine.py:351-390) plus the accumulator fold of the same nodes (centrality.py:132-150,
    one thread like the reference's numpy observer).  Returns a list of (arcs, seconds)."""
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
    sum_dist = np.zeros(n, np.float64)
    sum_recip = np.zeros(n, np.float64)
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    Pd = lambda a, k: ctypes.c_void_p(a.ctypes.data + 8 * k)  # noqa: E731

    def run_range(lo, hi):
        # arc-balanced sub-ranges over `threads` pthreads, like engine.py:351-390, then
        # the accumulate of the same rows (t = 1)
        t0 = time.perf_counter()
        L.orc_iterate_range_mt(lo, hi, P(off), P(suc), P(cur), P(nxt), P(chg_prev),
                               P(chg_now), P(est), P(new_est), b, 1, threads)
        L.orc_accumulate(hi - lo, 1, Pd(est, lo), Pd(new_est, lo), Pd(sum_dist, lo),
                         Pd(sum_recip, lo))
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


def bench_config(cfgd, n: int, m: int, world: int = 1, exchange: str = "push") -> dict:
    """The workload description both arms print (identical, so the driver can pair them)."""
    p = 1 << cfgd.log2m
    return {"workload": f"{cfgd.name}: {cfgd.description}", "n": n, "m": m,
            "log2m": cfgd.log2m, "register_width": 5, "hash_seed": cfgd.hash_seed,
            "step": "one dense iteration (all sources changed): union + estimate + "
                    "accumulate for %s" % "/".join(cfgd.outputs),
            "l2": ("inputs larger than L2 (%.2f GB of registers + %.2f GB of CSR), no flush"
                   if n * p > 126e6 else
                   "registers (%.2f GB) + CSR (%.2f GB) partly L2-resident, no flush: a "
                   "small-graph line") % (n * p / 1e9, (8 * (n + 1) + 4 * m) / 1e9),
            "parallelism": (f"node-partition x{world}, {exchange} exchange"
                            if world > 1 else "single GPU")}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1308_2144_b200 import _lib
    # the graph is built by the oracle library's copy of the builders: this process maps
    # no product library (only oracle/liborc.so)
    _lib.use_graph_library(os.path.join(REPO, "oracle", "liborc.so"))
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
        "config": bench_config(cfg, g.n, g.m, args.gpus, args.exchange),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{len(timed)} dense-step samples (union pass of "
                                   f"hll_union_range restated in C on {threads} pthreads + "
                                   f"the accumulate of the same rows), ~{per_step:.1f} s each, "
                                   f"{arcs} arcs total; " + _local_sub_csr_note()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "mapped_repo_libs": mapped_repo_libs(),
    }
    pkg = None if args.no_reference_package else reference_package_sample(g, cfg, threads)
    if pkg is not None:
        line["reference_package"] = pkg
    print(json.dumps(line), flush=True)


def reference_package_sample(g, cfgd, threads: int):
    """The reference package itself (numba kernels, hyperball from baseline/_ref -- the one
    offline install of /root/reference/pkg) on the same graph: initialize, one untimed
    iteration (numba compile), then two timed dense iterations of its own iterate()
    (engine.py:362-399) with a CentralityAccumulator and os.cpu_count() workers.  Reported
    beside the arm's value (the C port, which runs at or above numba speed) for
    transparency; None when the package is not installed."""
    path = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "hyperball")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_hb_bench")
    sys.path.insert(0, path)
    try:
        import hyperball as ref
    except Exception as exc:                       # numba missing etc.
        return {"unavailable": repr(exc)[:200]}
    gT = ref.CsrGraph(np.asarray(g.offsets, np.int64), np.asarray(g.successors, np.int64))
    cfg = ref.HyperBallConfig(params=ref.CounterParams(b=cfgd.log2m, seed=cfgd.hash_seed),
                              workers=threads)
    acc = ref.CentralityAccumulator(gT.n)
    st = ref.initialize(gT, cfg)
    ref.iterate(gT, st, [acc])                     # warm-up: numba compiles / loads here
    secs, arcs = 0.0, 0
    for _ in range(2):
        t0 = time.perf_counter()
        ref.iterate(gT, st, [acc])
        secs += time.perf_counter() - t0
        arcs += gT.m                               # iterations 2-3: (nearly) every source
    p = 1 << cfgd.log2m                            # changed, every arc merged
    return {"value": arcs * p / secs, "unit": UNIT, "cores": threads,
            "kind": "reference package (numba)",
            "sample": f"iterations 2 and 3 of hyperball.iterate on the whole graph "
                      f"({gT.m} arcs each), {threads} workers, CentralityAccumulator observer; "
                      f"{secs:.2f} s"}


# ------------------------------------------------------------------------ GPU arm

def load_traffic(config: str):
    """ncu DRAM bytes (read + write) per dense step of `config`, from the committed
    profile summary (profiles/ncu_traffic.json), or None."""
    tpath = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(tpath)).get(config)
    except Exception:
        return None


def dram_side(traffic, kernel_ms: float, peak: float) -> dict:
    """The DRAM side of the roofline: the ncu-measured bytes of one dense step (traffic,
    profiles/ncu_traffic.json) over the live kernel time -- what the HBM actually moved,
    next to `achieved` (algorithmic bytes, which count source rows the L2 served)."""
    if not traffic or not kernel_ms:
        return {}
    gbs = traffic / (kernel_ms * 1e-3) / 1e9
    return {"dram_gbs": gbs, "dram_frac": gbs / peak}


def dense_steps(g, cfgd, local: int, steps: int, warmup: int, schedule: str = "auto",
                world: int = 1, rank: int = 0, exchange: str = "push", clocks: bool = False):
    """Device-resident dense iterations of config `cfgd` on graph `g`: `warmup` untimed,
    then `steps` timed with CUDA events on the launching stream (barrier +
    synchronize on both sides; max over ranks).  Returns a dict of the measurements."""
    import torch
    import torch.distributed as dist

    import paper_1308_2144_b200 as hb
    from paper_1308_2144_b200 import _lib

    b, seed = cfgd.log2m, cfgd.hash_seed
    p = 1 << b
    n, m = g.n, g.m
    params = hb.CounterParams(b=b, seed=seed)
    cfg = hb.HyperBallConfig(params=params, device=local, schedule=schedule)
    acc = hb.CentralityAccumulator(n)
    rs = st = symm = comm = None
    if world > 1:
        from paper_1308_2144_b200.distributed import CudaRankState, TorchComm
        comm = TorchComm()
        rs = CudaRankState(g, cfg, world, rank)
        sums = rs.bind_sums()
        dev = rs.dev
        if exchange == "push":
            from paper_1308_2144_b200.distributed import setup_push
            symm = setup_push(rs)
    else:
        from paper_1308_2144_b200.engine import _bind_sums
        st = hb.initialize(g, cfg)
        dev = st._dev
        sums = _bind_sums(st, acc)
    s = dev.sched
    stream = dev.stream
    outputs = tuple(cfgd.outputs)
    need_dist = "closeness" in outputs or "lin" in outputs

    step_no = [0]

    def step(ev0=None, ev1=None):
        """One dense iteration: union kernels (+ exchange of changed rows when N > 1: fused
        into the union epilogue with --exchange push, else pack / all-gather / scatter)."""
        from paper_1308_2144_b200.distributed import _ptr_array
        import ctypes
        npeer, pn, pc, clear = 0, None, None, 1
        k_step = step_no[0]
        step_no[0] += 1
        if symm is not None:
            pnl, pcl = symm.peer_pointers(dev, k_step)     # inbox parity by step (packed)
            npeer, pn, pc, clear = len(pnl), _ptr_array(pnl), _ptr_array(pcl), 0
        if ev0 is not None:
            ev0.record(stream)
        _lib.union_step(_lib.StepArgs(
            n=n, lo=s.light_lo, hi=s.light_hi if dev.full_pass else s.light_hi_steady,
            offsets=s.offsets_ptr(), succ=s.succ.data_ptr(), cur=dev.cur.data_ptr(),
            nxt=dev.nxt.data_ptr(), chg_prev=dev.chg_prev.data_ptr(),
            chg_now=dev.chg_now.data_ptr(), est=dev.est.data_ptr(), b=b, dense=1,
            clear_chg_now=clear, t=1, lc_table=dev.lc.data_ptr(), alpha_p2=dev.alpha_p2,
            lc_cut=dev.lc_cut, sum_dist=sums.sum_dist.data_ptr() if need_dist else None,
            sum_recip=sums.sum_recip.data_ptr(), n_peers=npeer,
            peer_nxt=ctypes.cast(pn, ctypes.c_void_p) if pn is not None else None,
            peer_chg=ctypes.cast(pc, ctypes.c_void_p) if pc is not None else None,
            peer_packed_stride=symm.pstride if symm is not None else 0,
            nch_out=dev.counts.data_ptr(), merged_out=dev.counts.data_ptr() + 8,
            ticket=dev.ticket.data_ptr(), stream=stream.cuda_stream,
            **(dev.die_args() if symm is None else {}), **_lib.schedule_args(s)))
        if ev1 is not None:
            ev1.record(stream)
        nch, merged = (int(x) for x in dev.counts.cpu())   # the per-iteration termination read
        if symm is not None:
            # the all-reduce of the changed count is the barrier after which every peer's
            # pushed rows are visible; chg_prev stays all-ones so each step is iteration 1
            tot = torch.tensor([nch], dtype=torch.int64, device=dev.device)
            dist.all_reduce(tot)
            if symm.pstride:   # packed push: unpack the peers' rows (chg_prev is all ones)
                from paper_1308_2144_b200.distributed import unpack_inbox
                unpack_inbox(rs, symm.inbox_of(k_step), dev.chg_prev)
        elif rs is not None:
            rs.refresh_unowned()
            ids, rows, k = rs.gather_changed()
            _, parts = comm.exchange(ids, rows, k)
            for ids_q, rows_q in parts:
                rs.apply_remote(ids_q, rows_q)
        return nch, merged

    launches_per_step = (s.light_hi > s.light_lo) + (s.n_items > 0) + (s.n_heavy > 0) + (
        s.n_mega > 0 and s.n_heavy > s.n_mega)
    if world > 1 and symm is None:
        launches_per_step += 2 + (world - 1)   # refresh, gather, one scatter per peer
    elif symm is not None and symm.pstride:
        launches_per_step += 1                 # unpack of the peers' packed rows
    for _ in range(warmup):
        step()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    merged_check = None
    clk = ClockSampler(local) if clocks else None
    if clk is not None:
        clk.__enter__()
    t_start.record(stream)
    for i in range(steps):
        nch, merged = step(*evs[i])
        merged_check = merged
    t_end.record(stream)
    torch.cuda.synchronize()
    if clk is not None:
        clk.__exit__(None, None, None)
    if world > 1:
        dist.barrier()
    total_ms = t_start.elapsed_time(t_end)
    kernel_ms = [a.elapsed_time(b_) for a, b_ in evs]
    if world > 1:
        tt = torch.tensor([total_ms, sum(kernel_ms)], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms, ksum = tt.tolist()
        mt = torch.tensor([merged_check], dtype=torch.int64, device="cuda")
        dist.all_reduce(mt)
        merged_check = int(mt.item())
    else:
        ksum = sum(kernel_ms)
    assert merged_check == m, (merged_check, m)   # a dense step merges every arc
    ms_per_step = total_ms / steps
    k_ms = ksum / steps
    peak, peak_src = measured_peak()
    B = alg_bytes(n, m, p)
    achieved = B / world / (k_ms / 1000.0) / 1e9    # per GPU: its share of B / its kernel time
    out = {"ms_per_step": ms_per_step, "kernel_ms": k_ms, "value": m * p / (ms_per_step / 1e3),
           "alg_bytes": B, "achieved": achieved, "peak": peak, "peak_src": peak_src,
           "frac": achieved / peak, "launches_per_step": launches_per_step,
           "schedule": s.order, "heavy_nodes": s.n_heavy, "items": s.n_items,
           "clocks": clk.summary() if clk is not None else None}
    del st, rs, dev, sums, acc, symm
    return out


def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_1308_2144_b200 as hb
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
    outputs = tuple(cfgd.outputs)

    # ---------------------------------------------------------------- device-resident step
    d = dense_steps(g, cfgd, local, args.steps, args.warmup, args.schedule, world, rank,
                    args.exchange, clocks=True)
    torch.cuda.empty_cache()

    # ---------------------------------------------------------------- whole run + e2e
    def e2e_run(gp, what, h2d):
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
        dts = [r[0] for r in runs]
        merged_total, iters = runs[-1][1], runs[-1][2]
        if world > 1:
            tt = torch.tensor([sum(dts)], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            sum_dt = tt.item()
        else:
            sum_dt = sum(dts)
        mean_dt = sum_dt / len(dts)
        return {"value": merged_total * p / mean_dt, "unit": UNIT,
                "h2d_bytes_per_step": int(h2d),
                # the outputs and the 16-byte changed/merged counters read after every
                # iteration (the fused accumulator's final estimates stay on the device)
                "d2h_bytes_per_step": int(n * 8 * len(outputs) + 16 * iters),
                "seconds_per_run": mean_dt, "iterations": iters,
                "merged_arcs_per_run": merged_total,
                "what": "run(g, config, [CentralityAccumulator]) + finalize_{%s} from %s; "
                        "graph upload, schedule, seed, all iterations to convergence and "
                        "result download timed" % (",".join(outputs), what)}

    e2e = whole = e2e_ref_graph = None
    if not args.no_e2e:
        # pinned host copies of the graph: the user-side buffers of the e2e call
        off_pin = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
        suc_pin = torch.empty(m, dtype=torch.int32, pin_memory=True)
        hg = host_g()
        off_pin.numpy()[:] = hg.offsets
        suc_pin.numpy()[:] = hg.successors
        gp = hb.CsrGraph(off_pin.numpy(), suc_pin.numpy())
        e2e = e2e_run(gp, "pinned host CSR (int64 offsets, int32 ids)",
                      off_pin.numel() * 8 + suc_pin.numel() * 4)
        whole = {"iterations": e2e["iterations"], "merged_arcs": e2e["merged_arcs_per_run"],
                 "dense_equivalent_arcs": m * e2e["iterations"]}
        del gp, off_pin, suc_pin
        if not args.no_e2e_int64:
            # the reference's own input type: CsrGraph (graph.py:29-50) holds pageable int64
            # offsets and successors
            off64 = np.ascontiguousarray(hg.offsets, dtype=np.int64)
            suc64 = np.ascontiguousarray(hg.successors, dtype=np.int64)
            g64 = hb.CsrGraph(off64, suc64)
            e2e_ref_graph = e2e_run(g64, "the reference's CsrGraph layout (pageable int64 "
                                         "offsets and successors)",
                                    off64.nbytes + suc64.nbytes)
            del g64, off64, suc64
        torch.cuda.empty_cache()

    # ---------------------------------------------------------------- other configs
    per_config = None
    if rank == 0 and world == 1 and not args.no_per_config:
        per_config = {}
        if not args.no_cpu_baseline:
            host_g()                       # keep the host copy for the CPU baseline below
        g = None                           # a device-built graph frees its HBM here
        torch.cuda.empty_cache()
        for name in [c for c in args.per_config.split(",") if c and c != args.config]:
            try:
                cd = gen.CONFIGS[name]
                t0 = time.perf_counter()
                gq = cd.build_device(torch.device("cuda", local))
                torch.cuda.synchronize()
                log(f"[bench] per-config {name}: n={gq.n} m={gq.m} built in "
                    f"{time.perf_counter() - t0:.1f}s")
                r = dense_steps(gq, cd, local, args.per_config_steps, 3)
                pq = 1 << cd.log2m
                per_config[name] = {
                    "workload": f"{name}: {cd.description}", "n": gq.n, "m": gq.m,
                    "log2m": cd.log2m, "dense_ms": r["ms_per_step"],
                    "kernel_ms": r["kernel_ms"], "value": r["value"], "unit": UNIT,
                    "roofline": dict({"bound": "hbm", "achieved": r["achieved"], "peak": r["peak"],
                                      "unit": "GB/s", "frac": r["frac"],
                                      "algorithmic_bytes_per_launch": r["alg_bytes"],
                                      "traffic": load_traffic(name)},
                                     **dram_side(load_traffic(name), r["kernel_ms"], r["peak"])),
                    "schedule": r["schedule"], "steps": args.per_config_steps}
                del gq, r
                torch.cuda.empty_cache()
                log(f"[bench] per-config {name}: {per_config[name]['dense_ms']:.3f} ms, "
                    f"frac {per_config[name]['roofline']['frac']:.3f}")
            except Exception as exc:   # one config failing must not lose the headline line
                per_config[name] = {"error": repr(exc)[:300]}
                torch.cuda.empty_cache()

    # ---------------------------------------------------------------- CPU baseline
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        samples, _ = cpu_dense_sample(host_g(), b, seed, args.cpu_budget, threads, repeats=1)
        arcs, secs = samples[0]
        cpu = {"value": arcs * p / secs, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"one dense step (oracle/hb_oracle.c union pass on {threads} pthreads "
                         f"+ accumulate) over destination nodes holding {arcs} of {m} arcs "
                         f"({secs:.1f} s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": d["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": d["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic",
            "config": bench_config(cfgd, n, m, world, args.exchange),
            "schedule": {"order": d["schedule"], "heavy_nodes": d["heavy_nodes"],
                         "items": d["items"]},
            "roofline": {"bound": "hbm", "achieved": d["achieved"], "peak": d["peak"],
                         "unit": "GB/s", "frac": d["frac"], "traffic": load_traffic(args.config),
                         "algorithmic_bytes_per_launch": d["alg_bytes"],
                         **dram_side(load_traffic(args.config), d["kernel_ms"], d["peak"]),
                         "kernel_ms": d["kernel_ms"], "peak_source": d["peak_src"],
                         "kernels": "hb_union_step (light%s)" % (
                             " + heavy items + finish" if d["items"] else "")},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_reference_graph": e2e_ref_graph,
            "whole_run": whole,
            "per_config": per_config,
            "clocks": d["clocks"],
            "gpu_launches": d["launches_per_step"] * args.steps,
            "mapped_repo_libs": mapped_repo_libs(),
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
    ap.add_argument("--no-e2e-int64", action="store_true",
                    help="skip the second e2e from the reference's int64 CsrGraph")
    ap.add_argument("--per-config", default="config2,config3,config5",
                    help="other configs whose dense step is measured into per_config")
    ap.add_argument("--per-config-steps", type=int, default=10)
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0,
                    help="seconds of CPU work in the cpu_baseline sample")
    ap.add_argument("--no-reference-package", action="store_true",
                    help="--impl reference: skip timing the reference package (numba)")
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
