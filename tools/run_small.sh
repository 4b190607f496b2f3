#!/bin/bash
# small_f32 parity + A/B against the default pick on the stress points it covers.
# WLS overrides the workload list.
mkdir -p gpurun_out; : > gpurun_out/small.jsonl
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 2
timeout -s KILL 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "small_f32" > gpurun_out/pytest_small.log 2>&1; echo rc=$? >> gpurun_out/pytest_small.log
for wl in ${WLS:-stress_L192_S12_H96 stress_L336_S24_H96 stress_L720_S48_H96 stress_L1440_S96_H96 stress_L96_S12_H96}; do
  for v in small_f32 default ${EXTRA_V:-}; do
    ex=""; [ $v != default ] && ex="--variant $v"
    timeout -s KILL 120 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $ex > gpurun_out/sm.json 2> gpurun_out/sm.err
    python -c "import json; d=json.load(open('gpurun_out/sm.json')); print(json.dumps({'wl':'$wl','v':'$v','ms':round(d['ms_per_step'],4),'hbm':round(d['roofline']['frac'],4),'k':d['roofline']['kernel']}))" >> gpurun_out/small.jsonl 2>> gpurun_out/sm.err || echo "{\"wl\":\"$wl\",\"v\":\"$v\",\"error\":1}" >> gpurun_out/small.jsonl
  done
done
cat gpurun_out/small.jsonl
tail -3 gpurun_out/pytest_small.log
