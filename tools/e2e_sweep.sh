#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/e2e.jsonl
for ch in ${CHUNKS:-0 16 32 64 128}; do
  timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 --host-chunk $ch > gpurun_out/e.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e.json')); print(json.dumps({'chunk':$ch,'e2e':d['e2e']['value']}))" >> gpurun_out/e2e.jsonl
done
cat gpurun_out/e2e.jsonl
