#!/bin/bash
# One gpurun call: build, one ncu --set full capture of the forward on WL (default traffic),
# and its SASS source page as CSV (for tools/ncu_opmix.py / ncu_lines.py).  -> gpurun_out/
set -u
OUT=gpurun_out; mkdir -p $OUT
TAG=${TAG:-cur}
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 2; }
timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:prnet_fwd -s 2 -c 1 \
  -o $OUT/prof_$TAG -f python bench.py --workload ${WL:-traffic} ${VARIANT:+--variant $VARIANT} --profile --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > $OUT/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
ncu -i $OUT/prof_$TAG.ncu-rep --page source --csv --print-source sass > $OUT/src_$TAG.csv 2>/dev/null
ncu -i $OUT/prof_$TAG.ncu-rep --page raw --csv > $OUT/raw_$TAG.csv 2>/dev/null
ls -la $OUT | tail -5
echo done
