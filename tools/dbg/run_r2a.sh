python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_tcg_gpu.py tests/test_tcl_gpu.py -q -x -m gpu 2>&1 | tail -2
HS=720 STEPS=5 bash tools/stress_sweep.sh > /dev/null 2>&1; cat gpurun_out/stress.jsonl | grep -E "S12|error"
LIBS="libprnet.so libprnet_prev.so libprnet.so libprnet_prev.so" WLS="traffic" VARIANT=tc_quad bash tools/abl_tcl.sh
