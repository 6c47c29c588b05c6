make -s -C paper_1502_03917_b200/csrc > /dev/null 2>&1
timeout 120 python scripts/kbench.py --ops multicolour --iters 10 > gpurun_out/mc_kbench.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_p1_mc_sweep -c 1 \
  -o gpurun_out/mc_l12 -f python scripts/kbench.py --ops multicolour --iters 2 > gpurun_out/mc_ncu.log 2>&1
