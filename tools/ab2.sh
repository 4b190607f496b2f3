#!/bin/bash
# A/B the working tree against .ab_prev/ (tools/ab_tree.sh): three alternating repetitions.
mkdir -p gpurun_out; : > gpurun_out/ab.jsonl
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2 3; do
  for side in new prev; do
    dir=.; [ $side = prev ] && dir=.ab_prev
    (cd $dir && timeout -s KILL 200 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e ${BENCH_EXTRA:-} > /tmp/ab.json 2>/dev/null)
    python -c "import json; d=json.load(open('/tmp/ab.json')); print(json.dumps({'side':'$side','rep':$rep,'ms':d['ms_per_step']}))" >> gpurun_out/ab.jsonl
  done
done
cat gpurun_out/ab.jsonl
