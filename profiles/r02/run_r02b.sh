set -x
mkdir -p gpurun_out/r02b
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/r02b/gputest.log 2>&1; echo rc=$? >> gpurun_out/r02b/gputest.log
timeout 400 python bench.py > gpurun_out/r02b/bench.json 2> gpurun_out/r02b/bench.err
timeout 600 python bench.py --emulate-gather 8 --link-gbs 770 --no-cpu-baseline > gpurun_out/r02b/bench_emu8.json 2> gpurun_out/r02b/bench_emu8.err
timeout 600 python bench.py --emulate-gather 2 --link-gbs 770 --no-cpu-baseline > gpurun_out/r02b/bench_emu2.json 2> gpurun_out/r02b/bench_emu2.err
