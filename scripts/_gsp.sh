cd $GRAFT_REPO_ROOT
python scripts/gs_small_prof.py 6 20 > gpurun_out/gsp_times.log 2>&1 || exit 1
python scripts/gs_small_prof.py 7 20 >> gpurun_out/gsp_times.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_p1_gs_small -s 5 -c 1 -o gpurun_out/gs_small_r01 python scripts/gs_small_prof.py 6 10 > gpurun_out/gsp_ncu.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_p1_gs_diag -s 5 -c 1 -o gpurun_out/gs_diag_r01 python scripts/gs_small_prof.py 7 10 >> gpurun_out/gsp_ncu.log 2>&1
