#!/bin/bash
# A/B: cp.async ring edges vs plain loads
python scripts/wf_debug.py 6 7 > gpurun_out/ab_async.log 2>&1
cp paper_1502_03917_b200/libocmg_b200_plain.so paper_1502_03917_b200/libocmg_b200.so
python scripts/wf_debug.py 6 7 > gpurun_out/ab_plain.log 2>&1
