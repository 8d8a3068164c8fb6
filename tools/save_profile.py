#!/usr/bin/env python
"""Copy the ncu evidence of one gpurun iteration into profiles/ (tracked):
  - launch list summary (per-kernel mean device time and share of the step), from launches_<tag>.csv
  - ncu --set full summary of the top kernel, from prof_<tag>.ncu-rep
  - profiles/traffic.json[<kernel>/<config>] = dram read+write bytes per launch (bench.py roofline.traffic)
usage: tools/save_profile.py <tag> <round> <config>
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def launches(tag, rnd, cfg):
    src = os.path.join(G, f"launches_{tag}.csv")
    rows = list(csv.reader(open(src)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(list)
    for d in data:
        agg[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    out = os.path.join(P, f"{rnd}_launches_{cfg}.txt")
    with open(out, "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 (cold-cache, serialised: compare shares)\n")
        f.write(f"# command: python bench.py --config {cfg} --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks\n")
        f.write(f"{'kernel':60s} {'launches':>8s} {'mean_us':>10s} {'share':>7s}\n")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"{k[:60]:60s} {len(v):8d} {sum(v) / len(v) / 1e3:10.1f} {sum(v) / tot:7.3f}\n")
    os.replace(src, src) if False else None
    subprocess.run(["cp", src, os.path.join(P, f"{rnd}_launches_{cfg}.csv")], check=True)
    print(open(out).read())


def full(tag, rnd, cfg):
    rep = os.path.join(G, f"prof_{tag}.ncu-rep")
    txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep], capture_output=True,
                         text=True).stdout
    name = txt.splitlines()[0].replace("## ", "").split("(")[0] if txt else "kernel"
    name = name.replace("void ", "").split("<")[0].split("::")[-1]   # template / namespace decorations
    with open(os.path.join(P, f"{rnd}_ncu_full_{name}_{cfg}.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none --import-source on -k regex:{name} -s 1 -c 1 (bench.py --config {cfg})\n")
        f.write(txt)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]

    def get(k):
        i = hdr.index(k)
        v = float(vals[i])
        u = units[i]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

    traffic = get("dram__bytes_read.sum") + get("dram__bytes_write.sum")
    tj = os.path.join(P, "traffic.json")
    d = json.load(open(tj)) if os.path.exists(tj) else {}
    d[f"{name}/{cfg}"] = {"dram_bytes_per_launch": traffic, "source": f"{rnd}_ncu_full_{name}_{cfg}.txt"}
    for key, metric in (("pipe_fma_pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                        ("pipe_alu_pct", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active")):
        if metric in hdr:
            d[f"{name}/{cfg}"][key] = float(vals[hdr.index(metric)])
    json.dump(d, open(tj, "w"), indent=1)
    print(txt)
    print("traffic", traffic)


if __name__ == "__main__":
    tag, rnd, cfg = sys.argv[1], sys.argv[2], sys.argv[3]
    if os.path.exists(os.path.join(G, f"launches_{tag}.csv")):
        launches(tag, rnd, cfg)
    if os.path.exists(os.path.join(G, f"prof_{tag}.ncu-rep")):
        full(tag, rnd, cfg)
