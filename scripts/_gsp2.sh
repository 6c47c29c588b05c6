cd $GRAFT_REPO_ROOT
for k in 3 4 5 6; do python scripts/gs_small_prof.py $k 200; done > gpurun_out/gsp_times.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "reference_mode or wavefront or unaligned or baseline_protocol or reference_protocol" > gpurun_out/gs_small_tests.log 2>&1
echo tests=$? >> gpurun_out/gs_small_tests.log
