#!/bin/bash
# Bench sweep over kernel variants / windows-per-CTA (tuning; one gpurun call).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
: > gpurun_out/sweep.jsonl
for cfg in ${SWEEP:-"mma_f16x3:0 tc_quad:0"}; do
  v=${cfg%%:*}; w=${cfg##*:}
  PRNET_WINDOWS_PER_CTA=$w timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --variant $v ${BENCH_EXTRA:-} > gpurun_out/sw.json 2> gpurun_out/sw.err
  rc=$?; [ $rc -eq 137 ] && { echo "timeout $cfg" >> gpurun_out/sweep.jsonl; exit 3; }
  python -c "import json,sys; d=json.load(open('gpurun_out/sw.json')); print(json.dumps({'variant':'$v','wpc':$w,'ms':d['ms_per_step'],'frac':d['roofline']['frac']}))" >> gpurun_out/sweep.jsonl 2>>gpurun_out/sw.err
done
cat gpurun_out/sweep.jsonl
