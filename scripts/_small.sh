for k in 2 3 4; do timeout 60 python scripts/small_sweep.py $k wavefront 50; done > gpurun_out/small.log 2>&1
timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv python scripts/small_sweep.py 2 wavefront 5 2>/dev/null | grep gpu__time | tail -3 >> gpurun_out/small.log
