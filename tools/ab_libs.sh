#!/bin/bash
# A/B timing of several prebuilt libprnet builds (LIBS) on several workloads (WLS), 3 alternating
# repetitions, one gpurun call -> gpurun_out/ab_libs.jsonl
set -u
OUT=gpurun_out; mkdir -p $OUT; : > $OUT/ab_libs.jsonl
for rep in ${REPS:-1 2 3}; do
  for wl in ${WLS}; do
    for lib in ${LIBS}; do
      PRNET_LIB=$PWD/paper_2404_02445_b200/$lib timeout -s KILL 200 python bench.py --workload $wl --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline --no-e2e > $OUT/abl.json 2>$OUT/abl.err
      python -c "import json; d=json.load(open('$OUT/abl.json')); print(json.dumps({'wl':'$wl','lib':'$lib','rep':$rep,'k':d['roofline'].get('kernel'),'ms':round(d['ms_per_step'],4)}))" >> $OUT/ab_libs.jsonl 2>>$OUT/abl_err.log
    done
  done
done
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/ab_libs.jsonl'):
    r=json.loads(l); d[(r['wl'],r['lib'])].append(r['ms'])
for k,v in sorted(d.items()): print(k, 'min %.4f'%min(v), 'all', v)
PY
