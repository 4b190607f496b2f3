#!/bin/bash
# Round-end evidence in one gpurun call: smoke, GPU tests, the default bench line
# (with e2e + cpu_baseline), the reference arm, a variant sweep, the ncu launch list
# and one full capture of the default kernel.  Fail-fast on a hang (rc 137).
set -u
mkdir -p gpurun_out
OUT=gpurun_out
step() { local t=$1 log=$2; shift 2; timeout -s KILL "$t" "$@" > "$log" 2>&1; local rc=$?; echo "rc=$rc" >> "$log"; [ $rc -eq 137 ] && { echo "TIMEOUT $*" >> $OUT/ABORTED; exit 3; }; return $rc; }
(nproc; free -g; lscpu | grep -E "Model name|^CPU\(s\)"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv) > $OUT/env.txt 2>&1
step 300 $OUT/build.log python -c "import __graft_entry__ as g; g.build()" || exit 2
step 120 $OUT/smoke.log python -c "import __graft_entry__ as g; g.smoke()" || exit 4
step 900 $OUT/pytest_gpu.log python -m pytest tests -m gpu -q
timeout -s KILL 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; [ $? -eq 137 ] && exit 3
timeout -s KILL 400 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; [ $? -eq 137 ] && exit 3
SWEEP="${SWEEP:-tc_quad:0 mma_f16x3:0 warp_f32:0}" step 600 $OUT/sweep.log ./tools/sweep.sh
for wl in ${EXTRA_WORKLOADS:-weather_h96 electricity stress_L720_S24_H96 stress_L1440_S24_H96 stress_L5760_S12_H96}; do
  timeout -s KILL 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_$wl.json 2> $OUT/bench_$wl.err; [ $? -eq 137 ] && exit 3
done
step 300 $OUT/ncu_launch_run.log ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --profile --steps 3 --warmup 2 --no-e2e --no-cpu-baseline
step 420 $OUT/ncu_full_run.log ncu --set full --clock-control none --import-source on -k regex:prnet_fwd -s 2 -c 1 \
    -o $OUT/prof_fwd -f python bench.py --profile --steps 1 --warmup 2 --no-e2e --no-cpu-baseline
echo done
