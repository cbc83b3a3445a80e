"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv) per kernel: launches, time,
share of the total, DRAM bytes.

  launch_summary.py list.csv title [frames [workload json]]

With `frames`, also prints the DRAM bytes per decoded frame of the decoder's
own kernels (channel generation and torch fills excluded); with `workload` and
`json`, stores that figure in the json file (bench.py's roofline.traffic)."""
import collections
import csv
import json
import os
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6,
         "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0}

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr, data = rows[hi], rows[hi + 1:]
ix = {h: i for i, h in enumerate(hdr)}
agg = collections.defaultdict(lambda: collections.defaultdict(float))
ids = collections.defaultdict(set)
for r in data:
    name = r[ix["Kernel Name"]]
    name = name.replace("(anonymous namespace)::", "").replace("ldpcb::", "")
    name = name.split("(")[0][:60]
    v = float(r[ix["Metric Value"]].replace(",", "")) * SCALE.get(r[ix["Metric Unit"]], 1.0)
    agg[name][r[ix["Metric Name"]]] += v
    ids[name].add(r[ix["ID"]])
total = sum(d["gpu__time_duration.sum"] for d in agg.values())
print(f"{sys.argv[2]} ncu launch list (cold-cache, serialised), total {total * 1e3:.2f} ms")
lib_bytes = 0.0
decode_kernels = []
for name, d in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
    t = d["gpu__time_duration.sum"]
    rd, wr = d["dram__bytes_read.sum"], d["dram__bytes_write.sum"]
    if "at::" not in name and "channel" not in name:
        decode_kernels.append(name)
        lib_bytes += rd + wr
    print(f"  {name:60s} launches {len(ids[name]):5d} time {t * 1e3:9.3f} ms ({t / total:6.1%}) "
          f"dram R {rd / 1e9:8.3f} GB W {wr / 1e9:7.3f} GB")
if len(sys.argv) > 3:
    per = lib_bytes / float(sys.argv[3])
    print(f"  decoder kernels: {per:.1f} DRAM bytes per frame ({sys.argv[3]} frames)")
    if len(sys.argv) > 5:
        path, wl = sys.argv[5], sys.argv[4]
        rec = json.load(open(path)) if os.path.exists(path) else {}
        rec[wl] = {"bytes_per_frame": round(per, 1), "kernels": sorted(set(decode_kernels)),
                   "source": f"{os.path.basename(sys.argv[1])}: ncu --metrics dram__bytes_read.sum,"
                             f"dram__bytes_write.sum, {sys.argv[3]} decoded frames"}
        json.dump(rec, open(path, "w"), indent=1)
