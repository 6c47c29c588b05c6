cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "multicolour or fused_coarse" > gpurun_out/mcs_tests.log 2>&1; echo tests=$? >> gpurun_out/mcs_tests.log
bash scripts/_wfl.sh multicolour
