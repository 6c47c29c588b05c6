# launch list of one exact-order L12 W-cycle at coarsest L1 (the first cycle is warm-up)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_wcycle_exact_l1.csv python scripts/wcycle_launches.py 12 w wavefront 1 > gpurun_out/wcyc.log 2>&1
echo rc=$? >> gpurun_out/wcyc.log
