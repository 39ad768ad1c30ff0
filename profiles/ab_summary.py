"""One line per bench run of gpurun_out/ab_libs.log (or argv[1]): tokens/s, clock, stage ms/layer."""
import json
import sys

for l in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab_libs.log"):
    name, js = l.split(" ", 1)
    try:
        d = json.loads(js)
    except Exception:
        print(name, "ERR", js[:100])
        continue
    st = d["stage_ms_per_layer"]
    print(f"{name:8s} {d['value'] / 1e3:7.1f}K clk {d['clocks']['sm_mhz']} g1 {st['gemm1_gateup_swiglu']:.3f} "
          f"g2 {st['gemm2_down']:.3f} comb {st['combine']:.3f} perm {st['permute']:.3f} router {st['router']:.3f}")
