# full GPU suite + config-3 solve timings
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
timeout 600 python scripts/solve_c3.py 12 1 3 > gpurun_out/solve_c3.log 2>&1; echo rc=$? >> gpurun_out/solve_c3.log
