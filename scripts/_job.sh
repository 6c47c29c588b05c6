for k in 7 8 10 12; do timeout 300 python scripts/mc_check.py $k; done > gpurun_out/mcd_check.log 2>&1
timeout 200 python scripts/kbench.py --ops multicolour > gpurun_out/mcd_ab.log 2>&1
