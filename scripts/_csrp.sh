cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "stokes" > gpurun_out/csrp_tests.log 2>&1; echo tests=$? >> gpurun_out/csrp_tests.log
timeout 1200 python bench.py --steps 3 --warmup 3 --no-solve-l12 --no-cpu > gpurun_out/csrp_bench.log 2>&1; echo bench=$? >> gpurun_out/csrp_bench.log
