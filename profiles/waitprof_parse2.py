"""GEMM_WAITPROF summary by launch order (printf lines arrive launch by launch): per launch of the
router / GEMM1 / GEMM2 sequence, the MMA thread's loop cycles and the fraction blocked on the stage
'full' barrier, the producer warps' fractions (stage-free wait, tile-id wait, TMA issue) and the
epilogue warps' (accumulator-full wait, tile-id wait, wait for the previous TMA store to read smem)."""
import sys
from collections import defaultdict

rows = defaultdict(list)
for line in open(sys.argv[1]):
    f = line.split()
    if f and f[0] in ("WPM", "WPP", "WPE"):
        rows[f[0]].append([int(v) for v in f[1:]])
names = ["router", "gemm1", "gemm2"]
nm = len(rows["WPM"]) // 9 if rows["WPM"] else 0
for tag, per in (("WPM", 74), ("WPP", 296), ("WPE", 148)):
    r = rows[tag]
    for i in range(len(r) // per):
        ch = r[i * per:(i + 1) * per]
        if tag == "WPM":
            tot = sum(c[1] for c in ch)
            print(f"{names[i % 3]:7s} it{i // 3} MMA   cycles {tot / len(ch):.3g} full {sum(c[2] for c in ch) / tot:.3f} "
                  f"A {sum(c[3] for c in ch) / tot:.3f} acc {sum(c[4] for c in ch) / tot:.3f} ring {sum(c[5] for c in ch) / tot:.3f}")
        elif tag == "WPP":
            tot = sum(c[2] for c in ch)
            print(f"{names[i % 3]:7s} it{i // 3} PROD  cycles {tot / len(ch):.3g} empty {sum(c[3] for c in ch) / tot:.3f} "
                  f"sched {sum(c[4] for c in ch) / tot:.3f} issue {sum(c[5] for c in ch) / tot:.3f}")
        else:
            tot = sum(c[2] for c in ch)
            print(f"{names[i % 3]:7s} it{i // 3} EPI   cycles {tot / len(ch):.3g} tfull {sum(c[3] for c in ch) / tot:.3f} "
                  f"ring {sum(c[4] for c in ch) / tot:.3f} store-read {sum(c[5] for c in ch) / tot:.3f}")
