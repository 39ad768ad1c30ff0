#!/bin/bash
# Session 4: tile rasterisation of the grouped GEMMs (ASYNCEP_GEMM_RASTER = G row tiles walked
# row-first; 0 = row-tile-major, the default), materialised dispatch, one 235B layer at 32K tokens:
# ncu duration and SM cycles (clock-independent) of GEMM1 / GEMM2, BF16 and FP8, two rounds.
O=gpurun_out/s4raster; mkdir -p $O
M=gpu__time_duration.sum,sm__cycles_elapsed.max,dram__bytes_read.sum,lts__t_sector_hit_rate.pct
for round in 1 2; do
  for d in bf16 fp8; do
    F=""; [ $d = fp8 ] && F="--fp8"
    for r in 0 2 4 8 16; do
      ASYNCEP_GEMM_RASTER=$r timeout 300 ncu --metrics $M --clock-control none -k regex:gemm_tc_kernel -s 3 -c 3 --csv \
        --log-file $O/${d}_r${r}_${round}.csv python profiles/prof_layer.py --iters 2 $F > /dev/null 2>&1
    done
  done
done
