#!/bin/bash
# lane_f32 bring-up: its parity tests, tc_long floor tests, then A/B on the small-N stress points
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_lane_gpu.py tests/test_tcl_gpu.py -m gpu -x -q -p no:cacheprovider > gpurun_out/lane_tests.log 2>&1; echo "lane+tcl rc=$?"; tail -15 gpurun_out/lane_tests.log
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -p no:cacheprovider -k "low_seasonal or lane or sliding or long_lookback" > gpurun_out/par_tests.log 2>&1; echo "par rc=$?"; tail -3 gpurun_out/par_tests.log
WLS="${WLS:-stress_L96_S24_H96 stress_L96_S48_H96 stress_L96_S96_H96 stress_L192_S48_H96 stress_L192_S96_H96 stress_L336_S96_H96 stress_L96_S24_H720 stress_L96_S48_H720 stress_L192_S96_H720 etth1}" VARIANTS="auto lane_f32" bash tools/ab_var.sh 2>&1 | tail -25
TAG=lane24 WL=stress_L96_S24_H96 VARIANT=lane_f32 bash tools/prof_opmix.sh > /dev/null 2>&1
python tools/rawkeys.py gpurun_out/raw_lane24.csv | head -30
