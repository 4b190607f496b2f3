#!/bin/bash
# Full GPU test suite + smoke + widened-mode bench lines (one gpurun call).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 2
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1; echo rc=$? >> gpurun_out/pytest_all.log
for opt in "--metric-variant 1" "--metric-variant 2" "--instance-norm" "--metric-variant 3 --instance-norm"; do
  tag=$(echo $opt | tr -d ' -')
  timeout -s KILL 300 python bench.py $opt --steps 20 --warmup 3 --no-e2e > gpurun_out/bench_wide_$tag.json 2> gpurun_out/bench_wide_$tag.err
done
