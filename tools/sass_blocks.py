"""Group an ncu `--page source --csv --print-source sass` dump into straight-line blocks
(runs of equal execution count) and print each block's share of instructions and stall
samples with its top opcodes.   usage: python tools/sass_blocks.py dump.csv [min_share%]"""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iexe, ism = (hdr.index("Address"), hdr.index("Source"),
                       hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"))
body = [r for r in rows[2:] if len(r) > iexe]
tot = sum(int(r[iexe]) for r in body)
tots = sum(int(r[ism]) for r in body)
print(f"total {tot} warp instructions, {tots} stall samples")
blocks, cur = [], None
for k, r in enumerate(body):
    e = int(r[iexe])
    if cur is None or e != cur["exec"]:
        cur = {"start": k, "exec": e, "n": 0, "inst": 0, "smp": 0, "ops": collections.Counter()}
        blocks.append(cur)
    cur["n"] += 1
    cur["inst"] += e
    cur["smp"] += int(r[ism])
    op = r[isrc].split()[0] if r[isrc].split() else "?"
    if op.startswith("@"):
        op = r[isrc].split()[1]
    cur["ops"][op.split(".")[0]] += 1
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
for b in blocks:
    if 100 * b["inst"] / tot >= thr or 100 * b["smp"] / max(tots, 1) >= thr:
        print(f"@{b['start']:5d} n={b['n']:4d} exec={b['exec']:11d} inst {100*b['inst']/tot:5.1f}% "
              f"stall {100*b['smp']/max(tots,1):5.1f}%  {dict(b['ops'].most_common(8))}")
