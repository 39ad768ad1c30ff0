#!/bin/bash
# A/B of grouped-GEMM variants on one box: ncu per-kernel cycles, DRAM bytes, tensor-pipe %.
# usage: bash profiles/ab_gemm.sh NCTA,RASTER ...   (csv files land in gpurun_out/ab_*.csv)
M=gpu__time_duration.sum,sm__cycles_elapsed.max,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second
mkdir -p gpurun_out
# each argument: NCTA,RASTER,POL_A,POL_B   (policy 0 normal, 1 evict_last, 2 evict_first)
for cfg in "$@"; do
  IFS=, read n r pa pb pr <<< "$cfg"
  ASYNCEP_L2_PROMO=${pr:-256} ASYNCEP_GEMM_NCTA=$n ASYNCEP_GEMM_RASTER=$r ASYNCEP_POL_A=$pa ASYNCEP_POL_B=$pb timeout 300 ncu --metrics $M --clock-control none -k regex:"gemm_tc_kernel" -s 3 -c 2 --csv --log-file gpurun_out/ab_${n}_${r}_${pa}_${pb}_${pr:-256}.csv python profiles/prof_layer.py --iters 2 > /dev/null 2>&1
done
