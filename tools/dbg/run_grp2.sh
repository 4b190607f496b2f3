#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_grp_gpu.py tests/test_parity_gpu.py -k "grp or small or short or etth1" -m gpu -x -q -p no:cacheprovider > gpurun_out/grp_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/grp_tests.log
WLS="stress_L96_S12_H96 stress_L96_S24_H96 stress_L192_S12_H96 stress_L96_S48_H96 stress_L96_S96_H96 stress_L192_S48_H96 stress_L336_S48_H96 stress_L720_S96_H96 stress_L96_S48_H720 stress_L1440_S96_H96 etth1" VARIANTS="auto" bash tools/ab_var.sh 2>&1 | tail -12
