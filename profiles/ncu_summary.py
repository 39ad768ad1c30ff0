#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run here, on the CPU box, from gpurun_out/ files).

  python profiles/ncu_summary.py full   <rep.ncu-rep> <out.json>   # --set full capture
  python profiles/ncu_summary.py launch <launches.csv> <out.json>  # gpu__time_duration list
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
    "launch__block_size", "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__t_bytes.sum", "smsp__inst_executed.sum",
]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12, "ms": 1e-3, "us": 1e-6,
         "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "ns": 1e-9, "Ghz": 1e9, "Mhz": 1e6}


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for h, u, v in zip(hdr, units, vals):
            base = h.split(".", 1)[-1] if h.startswith(("TPC.", "SM_C.")) else h
            for key in KEYS:
                if h == key or h.endswith("." + key) or base == key:
                    try:
                        f = float(v.replace(",", ""))
                    except ValueError:
                        continue
                    d[key] = f * SCALE.get(u, 1.0) if u in SCALE else f
                    d[key + ".unit"] = "SI" if u in SCALE else u
        if "dram__bytes_read.sum" in d:
            d["dram_bytes_per_launch"] = d["dram__bytes_read.sum"] + d.get("dram__bytes_write.sum", 0.0)
        res.append(d)
    json.dump(res, open(out, "w"), indent=1)
    for d in res:
        print(json.dumps({k: v for k, v in d.items() if not k.endswith(".unit")}, indent=1))


def launch(path, out):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("(anonymous namespace)::", "")
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-9 if r[ui] == "nsecond" else 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    res = sorted(({"kernel": k, "launches": n, "total_s": t, "share": t / tot} for k, (n, t) in agg.items()),
                 key=lambda d: -d["total_s"])
    json.dump({"total_s": tot, "kernels": res}, open(out, "w"), indent=1)
    for d in res:
        print(f"{d['share']*100:6.2f}%  {d['launches']:5d}  {d['total_s']*1e3:9.3f} ms  {d['kernel']}")


if __name__ == "__main__":
    {"full": full, "launch": launch}[sys.argv[1]](sys.argv[2], sys.argv[3])
