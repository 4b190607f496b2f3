#!/bin/bash
# One gpurun iteration: build, targeted GPU parity tests (K=<pytest -k expr>), an A/B of
# variants on one workload (VARIANTS, WL), and optionally (NCU=<variant>) one full ncu capture.
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo build failed; exit 2; }
if [ -n "${K:-}" ]; then
  timeout -s KILL ${TT:-600} python -m pytest tests -m gpu -q -x -k "$K" > $OUT/pytest_iter.log 2>&1
  echo "rc=$?" >> $OUT/pytest_iter.log; tail -5 $OUT/pytest_iter.log
fi
: > $OUT/ab.jsonl
for wl in ${WLS:-${WL:-traffic}}; do
for rep in 1 2; do
  for v in ${VARIANTS:-tc_quad}; do
    for lib in ${LIBS:-libprnet.so}; do
      PRNET_LIB=$PWD/paper_2404_02445_b200/$lib timeout -s KILL 200 python bench.py --workload $wl --variant $v --steps 20 --warmup 5 --no-cpu-baseline --no-e2e ${BENCH_EXTRA:-} > $OUT/ab_$v.json 2> $OUT/ab_$v.err
      python -c "import json; d=json.load(open('$OUT/ab_$v.json')); print(json.dumps({'wl':'$wl','v':'$v','lib':'$lib','rep':$rep,'ms':round(d['ms_per_step'],4),'frac':round(d['roofline']['frac'],4),'mhz':d.get('clocks',{}).get('sm_mhz')}))" >> $OUT/ab.jsonl 2>>$OUT/ab_err.log
    done
  done
done
done
cat $OUT/ab.jsonl
if [ -n "${NCU:-}" ]; then
  timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:prnet_fwd -s 2 -c 1 \
    -o $OUT/prof_$NCU -f python bench.py --workload ${WL:-traffic} --variant $NCU --profile --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > $OUT/ncu_$NCU.log 2>&1
  echo "ncu rc=$?"
fi
echo done
