timeout 1500 python -m pytest tests/test_fullsize_gpu.py -m gpu -q -x --durations=20 > gpurun_out/fullsize.log 2>&1; echo rc=$? >> gpurun_out/fullsize.log
