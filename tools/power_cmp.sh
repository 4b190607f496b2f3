#!/bin/bash
# Sustained bench of several variants back to back (clocks, power, ms per step).
mkdir -p gpurun_out; : > gpurun_out/power.jsonl
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in ${VARIANTS:-tc_quad mma_f16x3}; do
  timeout -s KILL 300 python bench.py --variant $v --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/pw.json 2> gpurun_out/pw.err
  python -c "import json; d=json.load(open('gpurun_out/pw.json')); print(json.dumps({'variant':'$v','ms':d['ms_per_step'],'clocks':d['clocks']}))" >> gpurun_out/power.jsonl
done
cat gpurun_out/power.jsonl
