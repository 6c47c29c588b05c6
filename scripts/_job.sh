for k in 7 9 10 12; do timeout 300 python scripts/mc_check.py $k; done > gpurun_out/mcd_check.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "multicolour or strip or fused or sweep_into or collapsed or rolling" > gpurun_out/mcd_tests.log 2>&1
python bench.py --quick --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
