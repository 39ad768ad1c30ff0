import csv, glob, io, sys
for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab_*.csv")):
    txt = open(f).read()
    rows = list(csv.reader(io.StringIO(txt[txt.find('"ID"'):])))
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = {}
    for r in rows[1:]:
        if len(r) > vi:
            per.setdefault((r[0], r[ki][:34]), {})[r[mi]] = r[vi]
    for (i, k), m in per.items():
        print(f.split("/")[-1], k, "ms=%s cyc=%s GHz=%s dramR=%s tens=%s L2hit=%s" % (
            m.get("gpu__time_duration.sum"), m.get("sm__cycles_elapsed.max"), m.get("sm__cycles_elapsed.avg.per_second"),
            m.get("dram__bytes_read.sum"), m.get("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
            m.get("lts__t_sector_hit_rate.pct")))
