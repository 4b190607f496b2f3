#!/bin/bash
# tensor-core head backward: parity, then timing against the FP32 kernel (PRNET_BWD_F32=1)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_backward_mma_gpu.py tests/test_backward_gpu.py tests/test_backward_full_gpu.py -m gpu -x -q -p no:cacheprovider > gpurun_out/bm_tests.log 2>&1; echo "tests rc=$?"; tail -25 gpurun_out/bm_tests.log | grep -v "^$" | tail -12
for wl in traffic electricity; do
  echo "$wl mma: $(timeout 300 python tools/bwd_time.py $wl 2>&1 | tail -1)"
  echo "$wl f32: $(PRNET_BWD_F32=1 timeout 300 python tools/bwd_time.py $wl 2>&1 | tail -1)"
done
echo "traffic full: $(timeout 300 python tools/bwd_time.py traffic --full 2>&1 | tail -1)"
