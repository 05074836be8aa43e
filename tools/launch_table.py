"""Summarise an ncu --csv launch list (gpu__time_duration, dram bytes) per kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, im, iv, iid = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
per = collections.defaultdict(dict)
for r in rows[1:]:
    per[int(r[iid])][r[im]] = float(r[iv].replace(",", ""))
    per[int(r[iid])]["name"] = r[ik]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in per.values():
    a = agg[d["name"].split("(")[0][:64]]
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0)
    a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
print(f"| kernel | launches | total ms | share | avg ms/launch | DRAM GB/launch |")
print("|---|---|---|---|---|---|")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    if a[1] / tot < 0.001:
        continue
    print(f"| `{k}` | {a[0]} | {a[1]/1e6:.2f} | {a[1]/tot*100:.1f}% | {a[1]/a[0]/1e6:.3f} | "
          f"{a[2]/a[0]/1e9:.3f} |")
