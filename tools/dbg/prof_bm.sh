#!/bin/bash
# ncu of the tensor-core head backward on Traffic (one launch)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:bwd_head_mma -s 1 -c 1 \
  -o gpurun_out/prof_bm -f python tools/bwd_time.py traffic > gpurun_out/ncu_bm.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/prof_bm.ncu-rep --page source --csv --print-source sass > gpurun_out/src_bm.csv 2>/dev/null
ncu -i gpurun_out/prof_bm.ncu-rep --page raw --csv > gpurun_out/raw_bm.csv 2>/dev/null
python tools/rawkeys.py gpurun_out/raw_bm.csv | head -30
