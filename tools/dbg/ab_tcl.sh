#!/bin/bash
# A/B of tc_long build flags (PRNET_TCL_NOZERO, PRNET_TCL_SLEEP_NS) on the long-lookback points
mkdir -p gpurun_out; : > gpurun_out/ab_tcl.jsonl
cd paper_2404_02445_b200
python _build.py lib_a.so > /dev/null 2>&1
python _build.py lib_b.so fwd_tcl.cu:-DPRNET_TCL_NOZERO=1 > /dev/null 2>&1
python _build.py lib_c.so fwd_tcl.cu:-DPRNET_TCL_SLEEP_NS=2000 > /dev/null 2>&1
python _build.py lib_d.so fwd_tcl.cu:-DPRNET_TCL_NOZERO=1 fwd_tcl.cu:-DPRNET_TCL_SLEEP_NS=2000 > /dev/null 2>&1
cd ..
for rep in 1 2; do
for wl in stress_L5760_S12_H96 stress_L2880_S12_H96 stress_L1440_S12_H96 stress_L5760_S24_H96 stress_L5760_S48_H96 stress_L720_S12_H720; do
  for lib in lib_a.so lib_b.so lib_c.so lib_d.so; do
    PRNET_LIB=$PWD/paper_2404_02445_b200/$lib timeout -s KILL 200 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print(json.dumps({'wl':'$wl','lib':'$lib','rep':$rep,'ms':round(d['ms_per_step'],3),'k':d['roofline']['kernel']}))" >> gpurun_out/ab_tcl.jsonl 2>/dev/null || echo "{\"wl\":\"$wl\",\"lib\":\"$lib\",\"err\":1}" >> gpurun_out/ab_tcl.jsonl
  done
done
done
cat gpurun_out/ab_tcl.jsonl
