cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/ -x -q -m gpu  > gpurun_out/pdl_tests.log 2>&1; echo tests=$? >> gpurun_out/pdl_tests.log
timeout 1200 python bench.py --steps 3 --warmup 3 --no-stokes-l10 --no-cpu > gpurun_out/pdl_bench.log 2>&1; echo bench=$? >> gpurun_out/pdl_bench.log
