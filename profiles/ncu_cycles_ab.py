"""Per-GEMM ncu SM cycles of A/B csv captures (ncu --metrics sm__cycles_elapsed.max,... --csv):
python profiles/ncu_cycles_ab.py 'gpurun_out/dir/*.csv' -> per (file tag, kernel) cycles, sorted."""
import csv
import glob
import io
import re
import sys
from collections import defaultdict

res = defaultdict(list)
for f in sorted(glob.glob(sys.argv[1])):
    tag = re.sub(r"_\d+\.csv$", "", f.split("/")[-1])
    txt = open(f).read()
    i = txt.find('"ID"')
    per = defaultdict(dict)
    for row in csv.DictReader(io.StringIO(txt[i:])):
        per[(int(row["ID"]), row["Kernel Name"])][row["Metric Name"]] = row["Metric Value"]
    for (kid, kn), m in sorted(per.items()):
        kind = "gemm1" if "<1," in kn else "gemm2" if "<0," in kn else "router"
        res[(tag, kind)].append(float(m["sm__cycles_elapsed.max"].replace(",", "")))
for k in sorted(res):
    v = res[k]
    print(f"{k[0]:14s} {k[1]:7s} " + " ".join(f"{x / 1e6:.4f}M" for x in v) + f"   mean {sum(v) / len(v) / 1e6:.4f}M")
