#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 2
timeout -s KILL 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "sliding" > gpurun_out/pytest_sl.log 2>&1; echo rc=$? >> gpurun_out/pytest_sl.log
timeout -s KILL 300 python bench.py --sliding --steps 20 --warmup 3 > gpurun_out/bench_sliding.json 2> gpurun_out/bench_sliding.err
timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err
