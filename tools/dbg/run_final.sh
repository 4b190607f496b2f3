#!/bin/bash
# Round-end evidence: GPU suite, smoke, default bench, stress sweep.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_suite.log 2>&1; echo "suite rc=$?" ; tail -3 gpurun_out/gpu_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json
HS="96 720" bash tools/stress_sweep.sh > /dev/null 2>&1; wc -l gpurun_out/stress.jsonl
