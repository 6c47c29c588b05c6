cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/ -x -q -m gpu > gpurun_out/final_tests.log 2>&1; echo tests=$? >> gpurun_out/final_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; echo rc=$? >> gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo rc=$? >> gpurun_out/bench_ref.err
python bench.py --quick > gpurun_out/bq.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_quick.csv python bench.py --quick > gpurun_out/ncu_l.log 2>&1
bash scripts/_wfl.sh multicolour; bash scripts/_wfl.sh wavefront
