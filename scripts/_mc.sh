timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "multicolour or strip or sweep_into or fused" > gpurun_out/mc.log 2>&1; echo rc=$? >> gpurun_out/mc.log
timeout 120 python scripts/kbench.py --ops multicolour --iters 20 >> gpurun_out/mc.log 2>&1
timeout 300 python bench.py --quick --steps 20 --warmup 5 --no-cpu > gpurun_out/mc_bench.json 2>&1
