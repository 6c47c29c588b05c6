# one ncu --set full capture of the exact-order sweep kernel (k_wavefront) at L10
make -s -C paper_1502_03917_b200/csrc > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_wavefront -c 1 \
  -o gpurun_out/wf_l12 -f python scripts/wf_time.py 12 > gpurun_out/wf_ncu.log 2>&1
echo rc=$? >> gpurun_out/wf_ncu.log
