#!/bin/bash
# windows-per-CTA sweep of the default kernel on WLS (one gpurun call) -> gpurun_out/wpc.jsonl
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 2
: > $OUT/wpc.jsonl
for wl in ${WLS}; do
  for w in ${WPCS:-0}; do
    PRNET_WINDOWS_PER_CTA=$w timeout -s KILL 120 python bench.py --workload $wl ${VA:-} --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/w1.json 2>$OUT/w1.err
    python -c "import json; d=json.load(open('$OUT/w1.json')); print(json.dumps({'wl':'$wl','wpc':$w,'k':d['roofline'].get('kernel'),'ms':round(d['ms_per_step'],4),'frac':round(d['roofline']['frac'],4)}))" >> $OUT/wpc.jsonl 2>>$OUT/wpc_err.log
  done
done
cat $OUT/wpc.jsonl
