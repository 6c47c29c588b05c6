cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "mid_levels or reference_mode or unaligned or wavefront_mode" > gpurun_out/gs_small_tests.log 2>&1
echo tests=$? >> gpurun_out/gs_small_tests.log
for k in 3 4 5 6 7 8; do timeout 60 python scripts/gs_small_prof.py $k 100; done > gpurun_out/gsp_times.log 2>&1
