#!/bin/bash
# One gpurun call: build, optional pytest (K=<-k expr> or TF=<test files>), then each workload in
# WLS x each variant in VARIANTS (auto = default pick), 20 timed steps -> gpurun_out/ab_var.jsonl
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 2; }
if [ -n "${TF:-}" ]; then
  timeout -s KILL ${TT:-900} python -m pytest $TF -m gpu -q -x ${K:+-k "$K"} > $OUT/pytest_iter.log 2>&1
  echo "pytest rc=$?" >> $OUT/pytest_iter.log; tail -4 $OUT/pytest_iter.log
fi
: > $OUT/ab_var.jsonl
for wl in ${WLS:-}; do
  for v in ${VARIANTS:-auto}; do
    va=""; [ "$v" != "auto" ] && va="--variant $v"
    timeout -s KILL 200 python bench.py --workload $wl $va --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline --no-e2e > $OUT/ab_one.json 2> $OUT/ab_one.err
    python -c "import json; d=json.load(open('$OUT/ab_one.json')); print(json.dumps({'wl':'$wl','v':'$v','k':d['roofline'].get('kernel'),'ms':round(d['ms_per_step'],4),'frac':round(d['roofline']['frac'],4),'mhz':d.get('clocks',{}).get('sm_mhz')}))" >> $OUT/ab_var.jsonl 2>>$OUT/ab_err.log || echo "{\"wl\":\"$wl\",\"v\":\"$v\",\"err\":\"$(tail -1 $OUT/ab_one.err | tr -d '"')\"}" >> $OUT/ab_var.jsonl
  done
done
cat $OUT/ab_var.jsonl
echo done
