#!/bin/bash
# One gpurun call: environment facts, smoke, GPU tests, a short bench, and the
# ncu launch list + one full capture of the forward kernel.  Outputs -> gpurun_out/.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
(nproc; free -g; lscpu | grep -E "Model name|^CPU\(s\)"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv) > $OUT/env.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python -m pytest tests -m gpu -q ${PYTEST_ARGS:--x} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
if [ "${NCU:-1}" = "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
      python bench.py --profile --steps 3 --warmup 2 --no-e2e --no-cpu-baseline ${NCU_BENCH_ARGS:-} > $OUT/ncu_launch_run.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:prnet_fwd -s 2 -c 1 \
      -o $OUT/prof_fwd -f python bench.py --profile --steps 1 --warmup 2 --no-e2e --no-cpu-baseline ${NCU_BENCH_ARGS:-} > $OUT/ncu_full_run.log 2>&1
fi
echo done
