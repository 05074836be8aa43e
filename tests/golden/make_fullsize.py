"""Reference-produced truth at BASELINE.json's full sizes (configs 1-4).

Run in the build container (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_fullsize.py [config2 ...]

For each config it builds the graph with ``paper_1308_2144_b200.generators`` (the same
bytes the GPU tests build; the graph digest is recorded), wraps it in the reference's own
``CsrGraph`` and drives the REFERENCE engine -- ``initialize`` + ``iterate`` with its numba
kernels on ``os.cpu_count()`` arc-balanced workers (engine.py:330-399) and a
``CentralityAccumulator`` -- recording after the seed and after every iteration the
chunked digest of ``register_matrix()`` (``reg_digest``), the sha256 of ``est`` and the
changed count, then the three finalizers' digests.  Output: tests/golden/fullsize.json
(small; the GPU tests compare against it).  Config 5 (2^32 arcs) does not fit this
container's memory in the reference's int64 CsrGraph; its GPU test uses the C oracle.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

sys.path.insert(0, HERE)
from digest import reg_digest  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run_config(name: str) -> dict:
    import hyperball as ref
    from paper_1308_2144_b200 import generators as gen
    cfgd = gen.CONFIGS[name]
    t0 = time.perf_counter()
    g = cfgd.build()
    digest = gen.graph_digest(g)
    gT = ref.CsrGraph(np.asarray(g.offsets, np.int64), np.asarray(g.successors, np.int64))
    del g
    workers = os.cpu_count() or 1
    cfg = ref.HyperBallConfig(params=ref.CounterParams(b=cfgd.log2m, seed=cfgd.hash_seed),
                              workers=workers)
    acc = ref.CentralityAccumulator(gT.n)
    st = ref.initialize(gT, cfg)
    regs, ests, nchs, secs = [reg_digest(st.register_matrix())], [sha(st.est)], [], []
    while True:
        t1 = time.perf_counter()
        nch = ref.iterate(gT, st, [acc])
        secs.append(time.perf_counter() - t1)
        nchs.append(int(nch))
        regs.append(reg_digest(st.register_matrix()))
        ests.append(sha(st.est))
        print(f"  {name} t={st.t} changed={nch} {secs[-1]:.2f}s", flush=True)
        if nch == 0:
            break
    acc.on_converged(st.est)
    out = dict(config=name, n=int(gT.n), m=int(gT.m), b=cfgd.log2m, seed=cfgd.hash_seed,
               graph_digest=digest, t=int(st.t), nch=nchs, reg_digests=regs,
               est_digests=ests, harmonic=sha(ref.finalize_harmonic(acc)),
               closeness=sha(ref.finalize_closeness(acc)), lin=sha(ref.finalize_lin(acc)),
               workers=workers, iterate_seconds=[round(s, 3) for s in secs],
               total_seconds=round(time.perf_counter() - t0, 1))
    return out


def main():
    names = sys.argv[1:] or ["config1", "config2", "config3", "config4"]
    path = os.path.join(HERE, "fullsize.json")
    have = json.load(open(path)) if os.path.exists(path) else {}
    for name in names:
        print(f"{name} ...", flush=True)
        have[name] = run_config(name)
        with open(path, "w") as fh:
            json.dump(have, fh, indent=1, sort_keys=True)
        print(f"{name}: t={have[name]['t']} in {have[name]['total_seconds']} s", flush=True)


if __name__ == "__main__":
    main()
