python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_grp_gpu.py -q -x -m gpu 2>&1 | grep -E "^E .*(Assert|Error)|passed|failed" | head -5
WLS="stress_L96_S12_H96 stress_L96_S24_H96 stress_L192_S24_H96 stress_L192_S12_H96 stress_L336_S24_H96 etth1 stress_L96_S12_H720 stress_L192_S24_H720" VARIANTS="auto group_f32" bash tools/ab_var.sh 2>&1 | grep wl
