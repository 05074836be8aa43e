"""Generate tests/golden/ fixtures by running the REFERENCE package itself.

Run in the build container (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports ``hyperball`` from /root/reference/pkg/src and, for every case below, drives
``initialize`` + ``iterate`` (engine.py:330-399) with a ``CentralityAccumulator``
(centrality.py:104-150) until no counter changes, recording after the seed and after
every iteration the sha256 of ``register_matrix()`` and of ``est`` plus the changed
count, then ``on_converged`` and the three finalizers (centrality.py:153-171).  Graphs
are the transpose the engine consumes: small hand-built ones are stored in
``arrays.npz``; generator-built ones are rebuilt by the tests from
``paper_1308_2144_b200.generators`` and checked against the stored digest.

Also pinned: hash values (hll.py:79-88), register values (hll.py:147-158), alpha and
estimator constants, the estimator on crafted rows including registers above 31
(_kernels.py:15-34), the packed ``HLLA`` blob (hll.py:290-295) and an ``HBCK``
checkpoint (engine.py:254-280).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import hyperball as ref  # noqa: E402
from hyperball import _kernels as ref_kernels  # noqa: E402
from hyperball.hll import POW2NEG, alpha, register_values  # noqa: E402

from paper_1308_2144_b200 import generators as gen  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------- forward graphs (G)
def path_graph(k):
    s = np.arange(k - 1)
    return ref.CsrGraph.from_edges(s, s + 1, n=k)


def cycle_graph(k):
    s = np.arange(k)
    return ref.CsrGraph.from_edges(s, (s + 1) % k, n=k)


def star_graph(k):
    return ref.CsrGraph.from_edges(np.zeros(k, np.int64), np.arange(1, k + 1), n=k + 1)


def complete_graph(k):
    s, d = np.meshgrid(np.arange(k), np.arange(k), indexing="ij")
    keep = s != d
    return ref.CsrGraph.from_edges(s[keep], d[keep], n=k)


def random_graph(seed, n, avg):
    rng = np.random.default_rng(seed)
    m = int(round(n * avg))
    if n == 0 or m == 0:
        return ref.CsrGraph(np.zeros(n + 1, np.int64), np.zeros(0, np.int64))
    return ref.CsrGraph.from_edges(rng.integers(0, n, m), rng.integers(0, n, m), n=n)


def random_dag(seed, n, avg):
    rng = np.random.default_rng(seed)
    m = int(round(n * avg))
    s, d = rng.integers(0, n, 2 * m), rng.integers(0, n, 2 * m)
    f = s < d
    return ref.CsrGraph.from_edges(s[f], d[f], n=n)


def islands(seed, n, avg):
    rng = np.random.default_rng(seed)
    half = n // 2
    parts = []
    for lo, hi in ((0, half), (half, n)):
        m = int(round((hi - lo) * avg))
        parts.append(lo + rng.integers(0, hi - lo, size=(2, m)))
    arcs = np.hstack(parts)
    return ref.CsrGraph.from_edges(arcs[0], arcs[1], n=n)


def empty_graph(n):
    return ref.CsrGraph(np.zeros(n + 1, np.int64), np.zeros(0, np.int64))


# (name, forward-graph builder or None, generator key or None, b, seed, width)
HAND = [
    ("path8", lambda: path_graph(8), [4, 6], [0, 42]),
    ("cycle5", lambda: cycle_graph(5), [4, 6, 12], [0]),
    ("star6", lambda: star_graph(6), [4, 7], [42]),
    ("complete7", lambda: complete_graph(7), [5, 8], [1]),
    ("random300", lambda: random_graph(7, 300, 3.0), [4, 5, 6, 7, 8, 9, 10], [42]),
    ("dag300", lambda: random_dag(8, 300, 2.0), [4, 6, 8], [42, 2**63 + 5]),
    ("islands400", lambda: islands(9, 400, 1.5), [4, 6, 11], [3]),
    ("sparse2000", lambda: random_graph(10, 2000, 1.1), [4, 6], [42]),
    ("empty0", lambda: empty_graph(0), [6], [42]),
    ("isolated5", lambda: empty_graph(5), [6], [42]),
    ("single1", lambda: empty_graph(1), [4], [0]),
]

GEN = [
    ("config1", lambda: gen.BUILDERS["config1"](), [6], [42]),
    ("config1_b4", lambda: gen.BUILDERS["config1"](), [4], [42]),
    ("rmat12", lambda: gen.rmat_t(12, 16 << 12, seed=11), [4, 7], [42]),
    ("disc14", lambda: gen.disconnected_t(1 << 14, 1 << 13, 0.1, 6.0, seed=12), [4, 6], [42]),
    ("web14", lambda: gen.weblike_t(1 << 14, seed=13, window=64), [8], [42]),
]

WIDTH_CASES = [  # register width variations (saturation at 2^w - 1)
    ("random300_w3", lambda: random_graph(7, 300, 3.0), 6, 42, 3),
    ("random300_w8", lambda: random_graph(7, 300, 3.0), 6, 42, 8),
]


WEIGHTED_CASES = [  # NodeWeights replicas (engine.py:100-119)
    ("random300", lambda: random_graph(7, 300, 3.0), 6, 42, 5, 1),
    ("islands400", lambda: islands(9, 400, 1.5), 8, 3, 5, 2),
    ("dag300", lambda: random_dag(8, 300, 2.0), 4, 42, 6, 3),
]


DISCOUNT_SPECS = [("harmonic", None), ("log", None), ("quad", None), ("const", None),
                  ("table", ((1.0, 0.5, 0.25), 0.125))]
DISCOUNT_CASES = [  # fused discounted-gain sums (centrality.py:26-101,149-150)
    ("random300", lambda: random_graph(7, 300, 3.0), 6, 42),
    ("sparse2000", lambda: random_graph(10, 2000, 1.1), 4, 42),
]


EXACT_CASES = [  # the exact bitset backend (engine.py:178-213, _kernels.py:117-172)
    # (name, builder, weights seed or None, with discounts)
    ("path8", lambda: path_graph(8), None, False),
    ("cycle5", lambda: cycle_graph(5), None, False),
    ("star6", lambda: star_graph(6), None, False),
    ("complete7", lambda: complete_graph(7), None, False),
    ("random300", lambda: random_graph(7, 300, 3.0), None, True),
    ("dag300", lambda: random_dag(8, 300, 2.0), None, False),
    ("islands400", lambda: islands(9, 400, 1.5), 2, False),
    ("random300", lambda: random_graph(7, 300, 3.0), 1, False),
    ("sparse2000", lambda: random_graph(10, 2000, 1.1), None, False),
    ("isolated5", lambda: empty_graph(5), None, False),
    ("single1", lambda: empty_graph(1), None, False),
    ("empty0", lambda: empty_graph(0), None, False),
]


def ref_discounts():
    out = []
    for name, tab in DISCOUNT_SPECS:
        if tab is None:
            out.append(ref.DiscountSpec.preset(name))
        else:
            out.append(ref.DiscountSpec.from_table(tab[0], tab[1], name="table"))
    return out


def drive(gT, b, seed, width=5, weights=None, discounts=(), backend="probabilistic"):
    cfg = ref.HyperBallConfig(params=ref.CounterParams(b=b, register_width=width, seed=seed),
                              workers=1, weights=weights, backend=backend)
    acc = ref.CentralityAccumulator(gT.n, discounts)
    state = ref.initialize(gT, cfg)
    regs, ests, nchs, clamps = [sha(state.register_matrix())], [sha(state.est)], [], 0
    if gT.n > 0:
        while True:
            old = state.est.copy()
            nch = ref.iterate(gT, state, [acc])
            clamps += int(((state.est - old) < 0).sum())
            regs.append(sha(state.register_matrix()))
            ests.append(sha(state.est))
            nchs.append(int(nch))
            if nch == 0:
                break
    acc.on_converged(state.est)
    final = dict(est=state.est.copy(), sum_dist=acc.sum_dist.copy(),
                 sum_recip=acc.sum_recip.copy(), coreach=acc.coreach.copy(),
                 closeness=ref.finalize_closeness(acc), harmonic=ref.finalize_harmonic(acc),
                 lin=ref.finalize_lin(acc))
    for spec in discounts:
        final[f"disc_{spec.name}"] = ref.finalize_discounted(acc, spec.name)
    return dict(t=int(state.t), nch=nchs, reg_digests=regs, est_digests=ests,
                negative_deltas=clamps), final, state


def main():
    cases, arrays = [], {}

    def add(name, gT, b, seed, width, stored, digest=None, weights=None, wseed=None,
            discounts=()):
        meta, final, state = drive(gT, b, seed, width,
                                   None if weights is None else ref.NodeWeights.from_values(weights),
                                   discounts)
        key = f"{name}_b{b}_s{seed % 1000}_w{width}" + ("" if wseed is None else f"_nw{wseed}")
        if discounts:
            key += "_disc"
            meta["discounts"] = [[nm, tab] for nm, tab in DISCOUNT_SPECS]
        meta.update(key=key, graph=name, n=int(gT.n), m=int(gT.m), b=b, seed=str(seed),
                    width=width, graph_stored=stored, graph_digest=digest,
                    weights_seed=wseed)
        if weights is not None:
            arrays[f"{key}/weights"] = np.asarray(weights, np.int64)
        for k, v in final.items():
            arrays[f"{key}/{k}"] = v
        cases.append(meta)
        print(f"{key}: n={gT.n} m={gT.m} t={meta['t']} nch={meta['nch']} "
              f"neg={meta['negative_deltas']}", flush=True)
        return state

    for name, build, bs, seeds in HAND:
        gT = ref.transpose(build())
        arrays[f"graph/{name}/offsets"] = np.asarray(gT.offsets, np.int64)
        arrays[f"graph/{name}/successors"] = np.asarray(gT.successors, np.int64)
        for b in bs:
            for s in seeds:
                add(name, gT, b, s, 5, True)
    for name, build, b, s, w in WIDTH_CASES:
        gT = ref.transpose(build())
        gname = name.split("_")[0]
        add(gname, gT, b, s, w, True)
    for name, build, b, s, w, wseed in WEIGHTED_CASES:
        gT = ref.transpose(build())
        wts = np.random.default_rng(wseed).integers(1, 6, gT.n)
        add(name, gT, b, s, w, True, weights=wts, wseed=wseed)
    for name, build, b, s in DISCOUNT_CASES:
        gT = ref.transpose(build())
        add(name, gT, b, s, 5, True, discounts=ref_discounts())
    for name, build, bs, seeds in GEN:
        g = build()
        digest = gen.graph_digest(g)
        gT = ref.CsrGraph(np.asarray(g.offsets, np.int64), np.asarray(g.successors, np.int64))
        for b in bs:
            for s in seeds:
                add(name, gT, b, s, 5, False, digest)

    exact_cases = []
    for name, build, wseed, with_disc in EXACT_CASES:
        gT = ref.transpose(build())
        wts = None if wseed is None else np.random.default_rng(wseed).integers(1, 6, gT.n)
        discs = ref_discounts() if with_disc else ()
        meta, final, _ = drive(gT, 6, 42, 5,
                               None if wts is None else ref.NodeWeights.from_values(wts),
                               discs, backend="exact")
        key = f"exact_{name}" + ("" if wseed is None else f"_nw{wseed}") + (
            "_disc" if with_disc else "")
        meta.update(key=key, graph=name, n=int(gT.n), m=int(gT.m), b=6, seed="42", width=5,
                    graph_stored=True, graph_digest=None, weights_seed=wseed,
                    backend="exact")
        if with_disc:
            meta["discounts"] = [[nm, tab] for nm, tab in DISCOUNT_SPECS]
        if wts is not None:
            arrays[f"{key}/weights"] = np.asarray(wts, np.int64)
        for k, v in final.items():
            arrays[f"{key}/{k}"] = v
        exact_cases.append(meta)
        print(f"{key}: n={gT.n} m={gT.m} t={meta['t']} nch={meta['nch']}", flush=True)

    # ---------------------------------------------------------------- pins
    pins = {}
    items = np.array([0, 1, 2, 3, 1000, 2**31 - 1, 2**40 + 7, 2**64 - 1], dtype=np.uint64)
    hashes = {}
    for seed in (0, 1, 42, 2**63 + 5, 2**64 - 1):
        for replica in (0, 1, 2, 17):
            hashes[f"{seed}:{replica}"] = [str(int(h)) for h in ref.hash_items(
                items, np.full(items.shape, replica, np.uint64), seed)]
    pins["hash_items"] = dict(items=[str(int(i)) for i in items], values=hashes)
    rv = {}
    rng = np.random.default_rng(5)
    hs = rng.integers(0, 2**63, 64, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    hs = np.concatenate([hs, np.array([0, 1, 2**64 - 1, 1 << 63, 15, 16], np.uint64)])
    for b in (4, 6, 8, 12):
        for w in (3, 5, 6, 8):
            idx, rho = register_values(hs, ref.CounterParams(b=b, register_width=w))
            rv[f"{b}:{w}"] = [idx.tolist(), rho.tolist()]
    pins["register_values"] = dict(hashes=[str(int(h)) for h in hs], values=rv)
    pins["alpha"] = {str(p): alpha(p) for p in (16, 32, 64, 128, 256, 512, 1024, 4096)}
    pins["alpha_p2"] = {str(p): alpha(p) * p * p for p in (16, 32, 64, 128, 256, 4096)}
    est_rows = {}
    for b in (4, 6, 7, 8, 12):
        p = 1 << b
        rows = [np.zeros(p, np.uint8)]
        one = np.zeros(p, np.uint8)
        one[3] = 1
        rows.append(one)
        rows.append(np.full(p, 31, np.uint8))
        rows.append(np.full(p, 61 - b, np.uint8))          # > 31: sequential-sum path
        rr = np.random.default_rng(b)
        for hi in (2, 6, 12, 32, 62):
            r = rr.integers(0, hi, p).astype(np.uint8)
            r[rr.random(p) < 0.3] = 0
            rows.append(r)
        for z in (1, p // 3, p - 1):                        # around the LC switch
            r = rr.integers(1, 4, p).astype(np.uint8)
            r[:z] = 0
            rows.append(r)
        R = np.stack(rows)
        out = np.zeros(len(rows))
        a2 = alpha(p) * p * p
        ref_kernels.estimate_register_rows(R, 0, len(rows), POW2NEG, a2, 2.5 * p, float(p), out)
        arrays[f"est_rows/{b}/rows"] = R
        arrays[f"est_rows/{b}/est"] = out
        est_rows[str(b)] = len(rows)
    pins["estimate_rows"] = est_rows
    dense = np.random.default_rng(3).integers(0, 32, (7, 64)).astype(np.uint8)
    pins["hlla_blob_w5"] = hashlib.sha256(ref.CounterArray.from_dense(
        dense, ref.CounterParams(b=6, register_width=5, seed=9)).to_blob()).hexdigest()
    pins["hlla_blob_w6"] = hashlib.sha256(ref.CounterArray.from_dense(
        dense, ref.CounterParams(b=6, register_width=6, seed=9)).to_blob()).hexdigest()
    arrays["hlla/dense"] = dense
    # HBCK checkpoint after 2 iterations of random300, b=6, seed=42
    gT = ref.transpose(random_graph(7, 300, 3.0))
    cfg = ref.HyperBallConfig(params=ref.CounterParams(b=6, seed=42))
    st = ref.initialize(gT, cfg)
    ref.iterate(gT, st)
    ref.iterate(gT, st)
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "ck.bin")
        st.save(path)
        pins["hbck_random300_b6_t2"] = hashlib.sha256(open(path, "rb").read()).hexdigest()
    # exact-kind HBCK (raw bitset rows + weights) after 2 iterations of weighted islands400
    gT = ref.transpose(islands(9, 400, 1.5))
    wts = ref.NodeWeights.from_values(np.random.default_rng(2).integers(1, 6, gT.n))
    cfg = ref.HyperBallConfig(params=ref.CounterParams(b=6, seed=42), weights=wts,
                              backend="exact")
    st = ref.initialize(gT, cfg)
    ref.iterate(gT, st)
    ref.iterate(gT, st)
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "ck.bin")
        st.save(path)
        pins["hbck_exact_islands400_nw2_t2"] = hashlib.sha256(
            open(path, "rb").read()).hexdigest()

    with open(os.path.join(HERE, "cases.json"), "w") as fh:
        json.dump(dict(cases=cases, exact_cases=exact_cases, pins=pins), fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "arrays.npz"), **arrays)
    print("wrote", len(cases), "cases")


if __name__ == "__main__":
    main()
