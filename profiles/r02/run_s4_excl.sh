#!/bin/bash
# Session 4: exclusive copy CTAs for the gather (ASYNCEP_GATHER_EXCL: 1024-thread CTAs with 120 KB of
# shared memory, only on the ASYNCEP_RESERVE_SMS SMs the GEMMs leave free) vs the default co-resident
# copy (one 128-thread CTA per SM beside the GEMMs), emulated N = 8 at the NVLink-5 rate; the bench's
# exposed_ag A/B (gathered vs two resident contexts, interleaved) in each run.
O=gpurun_out/s4excl; mkdir -p $O
run() {  # tag env... -- bench args
  tag=$1; shift
  env "$@" timeout 500 python bench.py --emulate-gather 8 --link-gbs 770 --steps 8 --warmup 3 --no-cpu-baseline $BARGS \
    > $O/$tag.json 2> $O/$tag.err
}
for T in 24576 32768; do
  for d in bf16 fp8; do
    BARGS="--tokens $T"; [ $d = fp8 ] && BARGS="$BARGS --fp8"
    run ${d}_${T}_coresident A=1
    run ${d}_${T}_excl8 ASYNCEP_RESERVE_SMS=8 ASYNCEP_GATHER_CTAS=8 ASYNCEP_GATHER_EXCL=120
    run ${d}_${T}_excl16 ASYNCEP_RESERVE_SMS=16 ASYNCEP_GATHER_CTAS=16 ASYNCEP_GATHER_EXCL=120
    run ${d}_${T}_coresident_b A=1
  done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/s4excl/*.json")):
    try:
        d = json.loads([x for x in open(f) if x.startswith("{")][-1]); e = d["exposed_ag"]
        print(f.split("/")[-1], round(d["value"]), "exp", round(e["frac_of_layer"], 4), "ctl",
              round(e.get("control", {}).get("frac_of_layer", 0), 4), "wait", round(e["wait_ms_per_layer"], 3),
              "res", round(e["step_ms_resident"], 2), "gat", round(e["step_ms_gathered"], 2), e.get("sm_mhz_per_leg"))
    except Exception as ex:
        print(f, "ERR", ex)
PY
