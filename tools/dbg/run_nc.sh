#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 500 python tools/dbg/tcl_nearconst.py 2>&1 | tail -12
TAG=lane24 WL=stress_L96_S24_H96 VARIANT=lane_f32 bash tools/prof_opmix.sh > /dev/null 2>&1
python tools/rawkeys.py gpurun_out/raw_lane24.csv | head -30
