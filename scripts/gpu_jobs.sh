#!/bin/bash
# The GPU jobs this repository's evidence came from, in one place (dev tool).
# Run on a B200 box from the repository root, e.g.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash scripts/gpu_jobs.sh evidence'
# Outputs go to gpurun_out/ (scratch); the summaries kept are copied into
# profiles/ by hand.
set -u
job=${1:-help}
mkdir -p gpurun_out
NVBASE="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false -Xcompiler -fPIC,-O2 -cudart static"
case "$job" in
  tests)      # full -m gpu suite, smoke()
    timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log ;;
  fullsize)   # BASELINE configs 2, 3, 5 against the reference's per-cycle fixtures
    timeout 1500 python -m pytest tests/test_fullsize_gpu.py -m gpu -q --durations=20 > gpurun_out/fullsize.log 2>&1; echo rc=$? >> gpurun_out/fullsize.log ;;
  evidence)   # bench line, reference arm, launch list, ncu of the two NE-GS kernels
    python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$? >> gpurun_out/bench.err
    python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo rc=$? >> gpurun_out/ref.err
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches.csv python bench.py --quick --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
    timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_wavefront -c 1 \
      -o gpurun_out/wf_l12 -f python scripts/wf_time.py 12 > gpurun_out/wf_ncu.log 2>&1
    timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_p1_mc_sweep -c 1 \
      -o gpurun_out/mc_l12 -f python scripts/kbench.py --ops multicolour --iters 2 > gpurun_out/mc_ncu.log 2>&1 ;;
  wavefront)  # exact-order sweep: timing + parity, then per-warp stage timers
    timeout 200 python scripts/wf_time.py 9 10 12 > gpurun_out/wf_time.log 2>&1
    (cd paper_1502_03917_b200/csrc && make -B NVFLAGS="$NVBASE -DOCMG_WF_PROFILE" > /dev/null 2>&1)
    timeout 120 python scripts/wf_prof.py 12 > gpurun_out/wf_prof12.log 2>&1
    make -B -C paper_1502_03917_b200/csrc > /dev/null 2>&1 ;;
  wfprofab)   # per-warp stage timers of WF_VARIANTS (profile build + extra flags)
    IFS=';' read -ra vs <<< "${WF_VARIANTS:-}"
    i=0
    for v in "${vs[@]}"; do
      (cd paper_1502_03917_b200/csrc && make -B NVFLAGS="$NVBASE -DOCMG_WF_PROFILE $v" > /dev/null 2>&1)
      echo "== variant [$v]" > gpurun_out/wfprof_v$i.log
      timeout 120 python scripts/wf_prof.py 12 >> gpurun_out/wfprof_v$i.log 2>&1
      cp gpurun_out/wfprof_k12.npy gpurun_out/wfprof_v$i.npy
      i=$((i+1))
    done
    make -B -C paper_1502_03917_b200/csrc > /dev/null 2>&1 ;;
  solves)     # config-3 solves at coarsest L1 and L3, both modes
    timeout 900 python scripts/solve_c3.py 12 1 3 > gpurun_out/solve_c3.log 2>&1 ;;
  wcycle)     # launch lists of one W-cycle at coarsest L1, both NE-GS modes
    for m in wavefront multicolour; do
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/wcycle_${m}_l1.csv python scripts/wcycle_launches.py 12 w $m 1 > gpurun_out/wcycle_$m.log 2>&1
    done ;;
  wfab)       # exact-order sweep A/B: WF_VARIANTS="flags1;flags2;..." (extra nvcc -D flags)
    IFS=';' read -ra vs <<< "${WF_VARIANTS:-}"
    for v in "${vs[@]}"; do
      (cd paper_1502_03917_b200/csrc && make -B NVFLAGS="$NVBASE $v" > /dev/null 2>&1)
      echo "== variant [$v]"
      timeout 200 python scripts/wf_time.py ${WF_LEVELS:-10 12} 2>&1 | grep sweep
    done > gpurun_out/wfab.log 2>&1
    make -B -C paper_1502_03917_b200/csrc > /dev/null 2>&1 ;;
  mc2)        # the experimental rolling-window multicolour kernel: parity, timing against
              # the default kernel, per-warp cycle counters (-DMC2_PROF build)
    for k in 7 8 10 12; do OCMG_MC_SWEEP=roll timeout 300 python scripts/mc_check.py $k; done > gpurun_out/mc2_check.log 2>&1
    { OCMG_MC_SWEEP=roll timeout 200 python scripts/kbench.py --ops multicolour | tail -1
      timeout 200 python scripts/kbench.py --ops multicolour | tail -1; } > gpurun_out/mc2_kbench.log 2>&1
    (cd paper_1502_03917_b200/csrc && make -B NVFLAGS="$NVBASE -DMC2_PROF" > /dev/null 2>&1)
    OCMG_MC_SWEEP=roll timeout 200 python scripts/mc2_prof.py 12 > gpurun_out/mc2_prof.log 2>&1
    make -B -C paper_1502_03917_b200/csrc > /dev/null 2>&1
    for m in micro_node micro_dfma_lat; do
      nvcc -O3 -std=c++17 --fmad=false -gencode arch=compute_100a,code=sm_100a -o /tmp/$m scripts/$m.cu && /tmp/$m
    done > gpurun_out/mc2_micro.log 2>&1 ;;
  micro)      # micro-benchmarks (built in place)
    for m in micro_lat micro_chain micro_wfchain micro_fp64; do
      nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --fmad=false -o scripts/$m scripts/$m.cu && ./scripts/$m
    done > gpurun_out/micro.log 2>&1 ;;
  *) echo "usage: bash scripts/gpu_jobs.sh {tests|fullsize|evidence|wavefront|solves|wcycle|wfab|mc2|micro}" ;;
esac
