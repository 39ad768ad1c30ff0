"""Summarise GEMM_WAITPROF printf lines: per kernel launch, the mean fraction of the loop
time each role spends blocked on a barrier (MMA: full / own-gathered-A / accumulator-free /
tile-id ring; producer and gather warps: stage-free)."""
import sys
from collections import defaultdict

segs, cur, seen = [], defaultdict(list), set()
for line in open(sys.argv[1]):
    f = line.split()
    if not f or f[0] not in ("WPM", "WPP", "WPG", "WPE"):
        continue
    key = (f[0], f[1], f[2] if f[0] != "WPM" else "")
    if key in seen:
        segs.append(cur)
        cur, seen = defaultdict(list), set()
    seen.add(key)
    cur[f[0]].append([int(v) for v in f[1:]])
segs.append(cur)
for i, s in enumerate(segs):
    out = [f"launch {i}:"]
    if s["WPM"]:
        n = len(s["WPM"])
        tot = sum(r[1] for r in s["WPM"]) / n
        fr = [sum(r[j] for r in s["WPM"]) / n / tot for j in (2, 3, 4, 5)]
        out.append(f"MMA x{n} cycles {tot:.3g} wait full {fr[0]:.3f} A {fr[1]:.3f} acc {fr[2]:.3f} ring {fr[3]:.3f}")
    for tag, name in (("WPP", "producer"), ("WPG", "gather")):
        if s[tag]:
            n = len(s[tag])
            tot = sum(r[2] for r in s[tag]) / n
            extra = f" sched {sum(r[4] for r in s[tag]) / n / tot:.3f}" if len(s[tag][0]) > 4 else ""
            if len(s[tag][0]) > 5:
                extra += f" issue {sum(r[5] for r in s[tag]) / n / tot:.3f}"
            out.append(f"{name} x{n} empty-wait {sum(r[3] for r in s[tag]) / n / tot:.3f}{extra}")
    if s["WPE"]:
        n = len(s["WPE"])
        tot = sum(r[2] for r in s["WPE"]) / n
        fr = [sum(r[j] for r in s["WPE"]) / n / tot for j in (3, 4, 5)]
        out.append(f"epilogue x{n} tfull {fr[0]:.3f} ring {fr[1]:.3f} store-read {fr[2]:.3f}")
    print("  ".join(out))
