O=gpurun_out/s4a; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_guard.py tests/test_gpu_asyncep.py tests/test_gpu_ipc.py -q -x > $O/new_tests.log 2>&1; echo "rc=$?" >> $O/new_tests.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -n 3 $O/new_tests.log $O/pytest_gpu.log
