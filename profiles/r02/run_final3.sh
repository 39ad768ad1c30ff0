# Round-2 validation + evidence run (one B200), third pass (round end).
O=gpurun_out/final3; mkdir -p $O
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > $O/clocks.csv &
SMI=$!
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > $O/gputest.log 2>&1; echo rc=$? >> $O/gputest.log
timeout 400 python bench.py > $O/bench_bf16.json 2> $O/bench_bf16.err
timeout 400 python bench.py --fp8 --no-cpu-baseline > $O/bench_fp8.json 2> $O/bench_fp8.err
timeout 400 python bench.py --shape 30b --no-cpu-baseline > $O/bench_30b.json 2> $O/bench_30b.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python bench.py --attn --no-cpu-baseline > $O/bench_attn.json 2> $O/bench_attn.err
for T in 8192 12288 16384 24576 32768 49152; do
  timeout 500 python bench.py --fp8 --emulate-gather 8 --link-gbs 770 --tokens $T --steps 6 --no-cpu-baseline >> $O/sweep_T_fp8.jsonl 2>> $O/sweep.err
done
timeout 500 python bench.py --emulate-gather 8 --link-gbs 770 --tokens 49152 --steps 6 --no-cpu-baseline >> $O/sweep_T_bf16.jsonl 2>> $O/sweep.err
timeout 500 python bench.py --emulate-gather 8 --link-gbs 770 --steps 10 --ab-steps 12 --no-cpu-baseline >> $O/sweep_T_bf16.jsonl 2>> $O/sweep.err
K='regex:gemm_tc_kernel|perm_hist|perm_scan|perm_scatter|combine_kernel|act_quant|quant_tokens|perm_quant|gather_copy'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 112 -c 224 --csv --log-file $O/launches_bf16.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/launch_bf16.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 144 -c 288 --csv --log-file $O/launches_fp8.csv python bench.py --fp8 --steps 2 --warmup 3 --no-cpu-baseline > $O/launch_fp8.log 2>&1
for f in "" "--fp8"; do
  n=bf16; [ -n "$f" ] && n=fp8
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:gemm_tc_kernel<\(int\)[01]' -s 2 -c 2 -o $O/gemm_full_$n python bench.py $f --layers 1 --steps 2 --warmup 3 --no-cpu-baseline --no-ab > $O/ncu_$n.log 2>&1
done
kill $SMI
