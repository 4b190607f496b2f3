#!/bin/bash
# A/B of tc_long builds (PRNET_LIB): LIBS on WLS -> gpurun_out/abl.jsonl (ablation builds: invalid numbers)
set -u
OUT=gpurun_out; mkdir -p $OUT; : > $OUT/abl.jsonl
for wl in ${WLS:-stress_L5760_S12_H96 stress_L720_S12_H96}; do
for lib in ${LIBS:-libprnet.so}; do
  PRNET_LIB=$PWD/paper_2404_02445_b200/$lib timeout -s KILL 200 python bench.py --workload $wl --variant ${VARIANT:-tc_long} --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ab_one.json 2> $OUT/ab_one.err
  python -c "import json; d=json.load(open('$OUT/ab_one.json')); print(json.dumps({'wl':'$wl','lib':'$lib','ms':round(d['ms_per_step'],4)}))" >> $OUT/abl.jsonl 2>>$OUT/ab_err.log
done; done
cat $OUT/abl.jsonl
