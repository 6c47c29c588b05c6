timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/fused.log 2>&1; echo rc=$? >> gpurun_out/fused.log
timeout 900 python -m pytest tests/test_fullsize_gpu.py -m gpu -q -x -k "c2 or c3" >> gpurun_out/fused.log 2>&1; echo rc=$? >> gpurun_out/fused.log
for k in 2 3; do timeout 60 python scripts/small_sweep.py $k wavefront 50; done >> gpurun_out/fused.log 2>&1
timeout 600 python scripts/solve_c3.py 12 1 > gpurun_out/solve_c3.log 2>&1; echo rc=$? >> gpurun_out/solve_c3.log
