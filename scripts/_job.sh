for k in 7 8 9 10 11 12; do timeout 300 python scripts/mc_check.py $k; done > gpurun_out/mcd_check.log 2>&1
timeout 200 python scripts/kbench.py --ops multicolour > gpurun_out/mcd_ab.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "multicolour or strip or fused or sweep_into or collapsed" > gpurun_out/mcd_tests.log 2>&1
