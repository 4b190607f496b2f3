#!/bin/bash
# One gpurun call: environment facts, smoke, GPU tests, a short bench, and the
# ncu launch list + one full capture of the forward kernel.  Outputs -> gpurun_out/.
# Fail-fast: a step killed by its timeout (rc 137, likely a hung kernel) stops
# the script so the box is never driven into gpurun's own limit.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
step() {  # step <seconds> <log> <cmd...>
  local t=$1 log=$2; shift 2
  timeout -s KILL "$t" "$@" > "$log" 2>&1
  local rc=$?
  echo "rc=$rc" >> "$log"
  if [ $rc -eq 137 ]; then echo "TIMEOUT in: $*" | tee -a $OUT/ABORTED; exit 3; fi
  return $rc
}
(nproc; free -g; lscpu | grep -E "Model name|^CPU\(s\)"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv) > $OUT/env.txt 2>&1
step 300 $OUT/build.log python -c "import __graft_entry__ as g; g.build()" || exit 2
step 120 $OUT/smoke.log python -c "import __graft_entry__ as g; g.smoke()" || { echo "smoke failed"; exit 4; }
if [ "${TESTS:-1}" = "1" ]; then
  step ${TEST_TIMEOUT:-900} $OUT/pytest_gpu.log python -m pytest tests -m gpu -q ${PYTEST_ARGS:--x}
fi
if [ "${BENCH:-1}" = "1" ]; then
  timeout -s KILL 400 python bench.py ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err
  rc=$?; echo "bench rc=$rc" >> $OUT/bench.err; [ $rc -eq 137 ] && exit 3
fi
if [ "${NCU:-1}" = "1" ]; then
  step 300 $OUT/ncu_launch_run.log ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
      python bench.py --profile --steps 3 --warmup 2 --no-e2e --no-cpu-baseline ${NCU_BENCH_ARGS:-}
  step 420 $OUT/ncu_full_run.log ncu --set full --clock-control none --import-source on -k regex:prnet_fwd -s 2 -c 1 \
      -o $OUT/prof_fwd -f python bench.py --profile --steps 1 --warmup 2 --no-e2e --no-cpu-baseline ${NCU_BENCH_ARGS:-}
fi
echo done
