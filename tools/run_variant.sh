#!/bin/bash
# One gpurun call for a kernel variant: build, its GPU parity tests, a bench line and
# (NCU=1) one full ncu capture of the forward kernel.  V=<variant> selects it.
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 2
V=${V:-tc_quad}
if [ "${TESTS:-1}" = 1 ]; then
  timeout -s KILL 300 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "$V" > $OUT/pytest_$V.log 2>&1
  echo "rc=$?" >> $OUT/pytest_$V.log
fi
timeout -s KILL 300 python bench.py --variant $V --steps 20 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_EXTRA:-} > $OUT/bench_$V.json 2> $OUT/bench_$V.err
if [ "${NCU:-1}" = 1 ]; then
  timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:prnet_fwd -s 2 -c 1 \
    -o $OUT/prof_$V -f python bench.py --variant $V --profile --steps 1 --warmup 2 --no-e2e --no-cpu-baseline ${BENCH_EXTRA:-} > $OUT/ncu_$V.log 2>&1
fi
echo done
