cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "reference_mode or wavefront or unaligned or baseline_protocol or reference_protocol or fixed_point or fused_coarse" > gpurun_out/gs_small_tests.log 2>&1
echo tests=$? >> gpurun_out/gs_small_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-stokes-l10 --no-cpu > gpurun_out/gs_small_bench.log 2>&1
echo bench=$? >> gpurun_out/gs_small_bench.log
bash scripts/_wfl.sh
