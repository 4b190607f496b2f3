#!/bin/bash
# End-of-round evidence in one gpurun call: build, smoke, GPU tests, the default bench line,
# the reference arm, other workloads, the ncu launch list + one full capture, the stress grid.
set -u
OUT=gpurun_out/final; mkdir -p $OUT
step() { local t=$1 log=$2; shift 2; timeout -s KILL "$t" "$@" > "$log" 2>&1; local rc=$?; echo "rc=$rc" >> "$log"; [ $rc -eq 137 ] && { echo "TIMEOUT $*" >> $OUT/ABORTED; exit 3; }; return $rc; }
(nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv) > $OUT/env.txt 2>&1
step 300 $OUT/build.log python -c "import __graft_entry__ as g; g.build()" || exit 2
step 120 $OUT/smoke.log python -c "import __graft_entry__ as g; g.smoke()" || exit 4
step 900 $OUT/pytest_gpu.log python -m pytest tests -m gpu -q
timeout -s KILL 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout -s KILL 400 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for wl in electricity weather_h96 weather_h192 weather_h336 weather_h720 etth1; do
  timeout -s KILL 300 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/bench_$wl.json 2> $OUT/bench_$wl.err
done
step 300 $OUT/ncu_launch_run.log ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --profile --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
step 420 $OUT/ncu_full_run.log ncu --set full --clock-control none --import-source on -k regex:prnet_fwd -s 3 -c 1 \
    -o $OUT/prof_fwd -f python bench.py --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline
bash tools/stress_sweep.sh > /dev/null 2>&1; cp gpurun_out/stress.jsonl $OUT/stress.jsonl
echo done
