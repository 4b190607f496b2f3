#!/bin/bash
# Traffic bench lines for every SURVEY 8(f) widening flag (final build).
mkdir -p gpurun_out/wide
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 2
run() { name=$1; shift; timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/wide/bench_wide_$name.json 2> gpurun_out/wide/$name.err; python -c "import json; d=json.load(open('gpurun_out/wide/bench_wide_$name.json')); print('$name', round(d['ms_per_step'],3), d['roofline']['kernel'], round(d['roofline']['frac'],3))"; }
run plain
run metricvariant1 --metric-variant 1
run metricvariant2 --metric-variant 2
run instancenorm --instance-norm
run metricvariant3instancenorm --metric-variant 3 --instance-norm
run component4 --metric-variant 4
run component7instancenorm --metric-variant 7 --instance-norm
run makernel25 --ma-kernel 25
run sliding --sliding
