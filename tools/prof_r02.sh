#!/bin/bash
# Round-2 evidence: default bench line (Traffic), its ncu launch list, ncu --set full captures of
# the new kernels on their stress points, the full-backward and BF16 timings -> gpurun_out/
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 2
timeout -s KILL 400 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_traffic.csv \
  python bench.py --profile --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for spec in "tcg96:stress_L2880_S96_H96:" "tcg12:stress_L336_S12_H96:" "tcl48:stress_L5760_S48_H96:" "tcl480:stress_L5760_S12_H96:tc_long" "tcq:traffic:"; do
  IFS=: read tag wl var <<< "$spec"
  timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:prnet_fwd -s 2 -c 1 \
    -o $OUT/prof_$tag -f python bench.py --workload $wl ${var:+--variant $var} --profile --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > $OUT/ncu_$tag.log 2>&1
done
python tools/bwd_time.py traffic --full > $OUT/bwd_full_traffic.json 2>&1
python tools/bwd_time.py traffic > $OUT/bwd_head_traffic.json 2>&1
python tools/bf16_time.py traffic > $OUT/bf16_traffic.json 2>&1
python tools/bf16_time.py electricity > $OUT/bf16_electricity.json 2>&1
ls $OUT
