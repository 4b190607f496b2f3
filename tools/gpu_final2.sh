#!/bin/bash
# Refresh after late kernel changes: GPU tests, default bench, the stress grid -> gpurun_out/final2
set -u
OUT=gpurun_out/final2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1 || exit 2
timeout -s KILL 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1
timeout -s KILL 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
bash tools/stress_sweep.sh > /dev/null 2>&1; cp gpurun_out/stress.jsonl $OUT/stress.jsonl
echo done
