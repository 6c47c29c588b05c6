timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_vanka_gpu.py -m gpu -q -x > gpurun_out/fused.log 2>&1; echo rc=$? >> gpurun_out/fused.log
timeout 600 python scripts/solve_c3.py 12 1 > gpurun_out/solve_c3.log 2>&1; echo rc=$? >> gpurun_out/solve_c3.log
