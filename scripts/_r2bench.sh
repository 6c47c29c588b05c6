# round-2 evidence: full bench, reference arm, launch list of the bench, ncu of k_wavefront
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo rc=$? >> gpurun_out/r02_bench.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r02_ref.json 2> gpurun_out/r02_ref.err; echo rc=$? >> gpurun_out/r02_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02_launches.csv python bench.py --quick --steps 3 --warmup 3 --no-cpu > gpurun_out/r02_ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_wavefront -c 1 \
  -o gpurun_out/r02_wf_l12 -f python scripts/wf_time.py 12 > gpurun_out/r02_wf_ncu.log 2>&1
