#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over tools/sanitize.py
mkdir -p gpurun_out/san
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 2
: > gpurun_out/san/san_summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 \
      python tools/sanitize.py > gpurun_out/san/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san/san_summary.txt
done
cat gpurun_out/san/san_summary.txt
