"""Fold the per-config ncu captures of tools/ncu_traffic.sh into profiles/ncu_traffic.json:
DRAM bytes (read + write) of the union kernels of the LAST dense step in each capture
(bench.py --steps 1 --warmup 3: four dense steps; the last one's launches are the ones
after the last k_light / k_heavy_partial boundary)."""
import collections
import csv
import json
import sys

out = json.load(open("profiles/ncu_traffic.json"))
for c in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f"gpurun_out/ncu_traffic_{c}.csv")) if len(r) > 10]
    hdr = rows[0]
    ik, im, iv, iid = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.OrderedDict()
    for r in rows[1:]:
        d = per.setdefault(int(r[iid]), {"name": r[ik].split("(")[0]})
        d[r[im]] = float(r[iv].replace(",", ""))
    launches = list(per.values())
    # one step = the launches from the last step-opening kernel on (heavy partial opens a
    # step when there are heavy items, else the light kernel)
    opener = "k_heavy_partial" if any("k_heavy_partial" in d["name"] for d in launches) else "k_light"
    start = max(i for i, d in enumerate(launches) if opener in d["name"])
    step = launches[start:]
    byts = sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in step)
    ms = sum(d["gpu__time_duration.sum"] for d in step) / 1e6
    out[c] = int(byts)
    out.setdefault("_kernels", {})[c] = {d["name"].replace("void ", ""): round(
        (d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]) / 1e9, 3) for d in step}
    print(c, f"{byts/1e9:.2f} GB DRAM in {ms:.3f} ms (ncu, serialised)", out["_kernels"][c])
out["_source"] = ("tools/ncu_traffic.sh: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
                  "--clock-control none -k regex:'k_light|k_heavy' on bench.py --config <c> --steps 1 "
                  "--warmup 3; bytes of the union kernels of the last dense step (tools/traffic_json.py)")
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
