O=gpurun_out/final4; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; echo rc=$? >> $O/gputest.log
timeout 400 python bench.py > $O/bench_bf16.json 2> $O/bench_bf16.err
timeout 400 python bench.py --fp8 --no-cpu-baseline > $O/bench_fp8.json 2> $O/bench_fp8.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
