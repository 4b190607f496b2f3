#!/bin/bash
# configs[4] stress grid: one bench line per (L, S) point (default kernel choice).
mkdir -p gpurun_out; : > gpurun_out/stress.jsonl
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for L in 96 192 336 720 1440 2880 5760; do for S in 12 24 48 96; do
  wl=stress_L${L}_S${S}_H96
  timeout -s KILL 120 python bench.py --workload $wl --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/st.json 2> gpurun_out/st.err
  python -c "import json; d=json.load(open('gpurun_out/st.json')); print(json.dumps({'wl':'$wl','N':d['config']['N'],'ms':round(d['ms_per_step'],4),'hbm_frac':round(d['roofline']['frac'],4),'alu_frac':round(d['roofline_alu']['frac'],4),'kernel':d['roofline']['kernel']}))" >> gpurun_out/stress.jsonl 2>>gpurun_out/st.err || echo "{\"wl\":\"$wl\",\"error\":1}" >> gpurun_out/stress.jsonl
done; done
cat gpurun_out/stress.jsonl
