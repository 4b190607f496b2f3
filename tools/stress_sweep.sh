#!/bin/bash
# configs[4] stress grid: one bench line per (L, S, H) point (default kernel choice), H in $HS.
mkdir -p gpurun_out; : > gpurun_out/stress.jsonl
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for H in ${HS:-96 720}; do
for L in 96 192 336 720 1440 2880 5760; do for S in 12 24 48 96; do
  wl=stress_L${L}_S${S}_H${H}
  timeout -s KILL 120 python bench.py --workload $wl --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/st.json 2> gpurun_out/st.err
  python -c "
import json; d=json.load(open('gpurun_out/st.json')); rc=d.get('roofline_compute') or d.get('roofline_alu') or {}
print(json.dumps({'wl':'$wl','N':d['config']['N'],'M':d['config']['M'],'ms':round(d['ms_per_step'],4),'hbm_frac':round(d['roofline']['frac'],4),'compute_frac':round(rc.get('frac',0),4),'compute_bound':rc.get('bound'),'kernel':d['roofline']['kernel']}))" >> gpurun_out/stress.jsonl 2>>gpurun_out/st.err || echo "{\"wl\":\"$wl\",\"error\":1}" >> gpurun_out/stress.jsonl
done; done; done
cat gpurun_out/stress.jsonl
