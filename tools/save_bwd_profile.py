#!/usr/bin/env python
"""ncu launch list of the backward (gpu__time_duration + dram bytes per kernel, tools/run_backward.py)
-> profiles/<round>_backward_<cfg>.txt and profiles/traffic.json["backward/<cfg>"] (measured DRAM
bytes per backward call; bench.py roofline_backward.dram).  usage: save_bwd_profile.py <csv> <round> <cfg>"""
import collections
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src, rnd, cfg = sys.argv[1], sys.argv[2], sys.argv[3]
txt = open(src).read()
txt = txt[txt.index('"ID"'):]
per = collections.OrderedDict()
for r in csv.DictReader(io.StringIO(txt)):
    k = (int(r["ID"]), r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", ""))
    per.setdefault(k, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * \
        {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}.get(r["Metric Unit"], 1)
# the backward = the last contiguous run of backward kernels (after the forward of run_backward.py)
names = ("keys_hist_kernel", "radix_hist_kernel", "radix_rowscan_kernel", "radix_scatter_kernel", "offsets_kernel",
         "seg_sort_grad_kernel", "grad_kernel")
items = [(k, v) for k, v in per.items() if k[1].split("::")[-1] in names]
# one backward call: from the last first-kernel (keys_hist: radix path; seg_sort: clouds <= 24576) to the end
start = max(i for i, (k, _) in enumerate(items) if k[1].endswith(("keys_hist_kernel", "seg_sort_grad_kernel")))
items = items[start:]
tot_t = sum(v.get("gpu__time_duration.sum", 0) for _, v in items) / 1e9
tot_b = sum(v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0) for _, v in items)
out = os.path.join(ROOT, "profiles", f"{rnd}_backward_{cfg}.txt")
with open(out, "w") as f:
    f.write(f"# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
            f"(tools/run_backward.py {cfg}; cold-cache, serialised)\n")
    f.write(f"{'kernel':40s} {'us':>9s} {'DRAM MB':>9s} {'GB/s':>8s}\n")
    for (i, n), v in items:
        t = v.get("gpu__time_duration.sum", 0) / 1e9
        b = v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
        f.write(f"{n.split('::')[-1]:40s} {t * 1e6:9.1f} {b / 1e6:9.1f} {b / t / 1e9 if t else 0:8.0f}\n")
    f.write(f"{'total':40s} {tot_t * 1e6:9.1f} {tot_b / 1e6:9.1f} {tot_b / tot_t / 1e9:8.0f}\n")
tj = os.path.join(ROOT, "profiles", "traffic.json")
d = json.load(open(tj)) if os.path.exists(tj) else {}
d[f"backward/{cfg}"] = {"dram_bytes_per_call": tot_b, "ms_cold": tot_t * 1e3, "source": os.path.basename(out)}
json.dump(d, open(tj, "w"), indent=1)
print(open(out).read())
