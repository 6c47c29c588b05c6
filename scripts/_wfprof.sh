# exact-order sweep: timing + parity (normal build), then per-warp stage
# timers (-DOCMG_WF_PROFILE build)
timeout 200 python scripts/wf_time.py 9 10 12 > gpurun_out/wf1.log 2>&1
cd paper_1502_03917_b200/csrc
make -B NVFLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false -Xcompiler -fPIC,-O2 -cudart static -DOCMG_WF_PROFILE" > /dev/null 2>&1
cd ../..
timeout 120 python scripts/wf_prof.py 10 > gpurun_out/wfp10.log 2>&1
timeout 120 python scripts/wf_prof.py 12 > gpurun_out/wfp12.log 2>&1
