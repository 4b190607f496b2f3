#!/bin/bash
# Quick GPU check of HEAD: build, smoke, GPU tests, default bench line, launch list, one full ncu capture.
set -u
OUT=gpurun_out; mkdir -p $OUT
step() { local t=$1 log=$2; shift 2; timeout -s KILL "$t" "$@" > "$log" 2>&1; local rc=$?; echo "rc=$rc" >> "$log"; [ $rc -eq 137 ] && { echo "TIMEOUT $*" >> $OUT/ABORTED; exit 3; }; return $rc; }
step 300 $OUT/build.log python -c "import __graft_entry__ as g; g.build()" || exit 2
step 120 $OUT/smoke.log python -c "import __graft_entry__ as g; g.smoke()" || exit 4
[ "${SKIP_TESTS:-0}" = 1 ] || step 900 $OUT/pytest_gpu.log python -m pytest tests -m gpu -q -x
timeout -s KILL 600 python bench.py ${BENCH_EXTRA:-} > $OUT/bench_default.json 2> $OUT/bench_default.err; [ $? -eq 137 ] && exit 3
[ "${SKIP_NCU:-0}" = 1 ] && exit 0
step 300 $OUT/ncu_launch_run.log ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --profile --steps 3 --warmup 2 --no-e2e --no-cpu-baseline ${BENCH_EXTRA:-}
step 420 $OUT/ncu_full_run.log ncu --set full --clock-control none --import-source on -k regex:prnet_fwd -s 2 -c 1 \
    -o $OUT/prof_fwd -f python bench.py --profile --steps 1 --warmup 2 --no-e2e --no-cpu-baseline ${BENCH_EXTRA:-}
echo done
