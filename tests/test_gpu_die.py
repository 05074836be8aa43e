"""Die-affine heavy items (hb_die_map, hb_die_partition, hb_step_args.die_head; DESIGN.md
section 9): the map itself, and bit-exact parity with the CPU oracle after every iteration
when the heavy items are merged in two passes by source die -- on graphs small enough for
the oracle, with HB_DIE_MIN_MB=0 lowering the size threshold so the path is taken."""

import ctypes
import hashlib

import numpy as np
import pytest

import oracle as orc

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_1308_2144_b200")
torch = pytest.importorskip("torch")
from paper_1308_2144_b200 import _lib, generators as gen  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def die_map(t):
    L = _lib.hb()
    words = int(L.hb_die_map_words(t.data_ptr(), t.numel()))
    bits = torch.zeros(words, dtype=torch.int32, device=t.device)
    stats = (ctypes.c_int64 * 4)()
    _lib.check(L.hb_die_map(t.data_ptr(), t.numel(), bits.data_ptr(), stats,
                            torch.cuda.current_stream().cuda_stream), "hb_die_map")
    return bits, [int(x) for x in stats], words


def test_die_map_splits_the_device(monkeypatch):
    monkeypatch.setenv("HB_DIE", "1")
    t = torch.full((64 << 20,), 7, dtype=torch.uint8, device="cuda:0")
    bits, stats, words = die_map(t)
    if stats[0] == 0:
        pytest.skip("device does not split into two L2 dies")
    chunks = (64 << 20) // 2048
    assert words * 32 >= chunks
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    assert 0.9 * sms <= stats[0] + stats[1] <= sms
    assert min(stats[0], stats[1]) * 4 >= stats[0] + stats[1]
    assert 0.2 * chunks < stats[2] < 0.8 * chunks        # about half of the chunks per die
    assert stats[3] < chunks // 10                       # the two latencies are far apart
    assert int((t != 7).sum()) == 0                      # the probe leaves the data alone
    # stable: a second measurement agrees on (nearly) every chunk
    bits2, stats2, _ = die_map(t)
    diff = (bits ^ bits2).cpu().numpy().view(np.uint32)
    assert sum(bin(int(w)).count("1") for w in diff[diff != 0]) < chunks // 10
    # unaligned base: chunk 0 is the 2 KB block holding base[0]
    u = t[1000:1000 + (8 << 20)]
    bits3, stats3, words3 = die_map(u)
    assert words3 == ((1000 + (8 << 20) + 2047) // 2048 + 31) // 32 and stats3[0] > 0
    b1 = np.unpackbits(bits.cpu().numpy().view(np.uint8), bitorder="little")
    b3 = np.unpackbits(bits3.cpu().numpy().view(np.uint8), bitorder="little")
    k = (8 << 20) // 2048
    assert (b1[:k] != b3[:k]).sum() < k // 10


@pytest.mark.parametrize("scale,b,width,frontier", [(14, 4, 5, False), (15, 5, 5, False),
                                                    (16, 4, 6, False), (15, 4, 5, True)])
def test_die_affine_items_vs_oracle(monkeypatch, scale, b, width, frontier):
    monkeypatch.setenv("HB_DIE", "1")
    monkeypatch.setenv("HB_DIE_MIN_MB", "0")
    g = gen.rmat_t(scale, 24 << scale, seed=21 + scale)
    off = np.asarray(g.offsets, np.int64)
    suc = np.asarray(g.successors, np.int64)
    want = orc.run_oracle(off, suc, b, 42, width=width, workers=4)
    cfg = hb.HyperBallConfig(params=hb.CounterParams(b=b, register_width=width, seed=42),
                             schedule="degree", frontier=frontier)
    acc = hb.CentralityAccumulator(g.n)
    st = hb.initialize(g, cfg)
    dev = st._dev if hasattr(st, "_dev") else st.dev
    regs, nchs = [sha(st.register_matrix())], []
    used = 0
    while True:
        used += bool(dev.die_args())
        nch = hb.iterate(g, st, [acc])
        regs.append(sha(st.register_matrix()))
        nchs.append(nch)
        if nch == 0:
            break
    if not dev.sched.die:
        pytest.skip("device does not split into two L2 dies")
    head, rows, split, stats = dev.sched.die
    assert rows > 0 and stats[0] > 0 and stats[1] > 0
    sp = split.cpu().numpy()
    assert sp.min() >= 0 and sp.max() <= dev.sched.item_arcs and 0 < sp.sum() < g.m
    # the path was taken (every step unless sparse iterations switch to frontier mode)
    assert dev.sched.n_items > 0 and (used > 0 if frontier else used == len(nchs))
    acc.on_converged(st.est)
    assert st.t == want.t and nchs == want.nch
    assert regs == want.reg_digests
    assert np.array_equal(hb.finalize_harmonic(acc).view(np.uint64),
                          want.harmonic.view(np.uint64))
