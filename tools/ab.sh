#!/bin/bash
# A/B timing of two builds of libprnet (PRNET_LIB) in one process sequence.
mkdir -p gpurun_out; : > gpurun_out/ab.jsonl
for rep in 1 2 3; do
  for lib in ${LIBS:-libprnet.so libprnet_prev.so}; do
    PRNET_LIB=$PWD/paper_2404_02445_b200/$lib timeout -s KILL 200 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e ${BENCH_EXTRA:-} > gpurun_out/ab.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print(json.dumps({'lib':'$lib','rep':$rep,'ms':d['ms_per_step']}))" >> gpurun_out/ab.jsonl
  done
done
cat gpurun_out/ab.jsonl
