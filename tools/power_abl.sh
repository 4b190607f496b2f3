for lib in libprnet.so libprnet_a1.so libprnet_a2.so libprnet.so; do
  PRNET_LIB=$PWD/paper_2404_02445_b200/$lib timeout -s KILL 200 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/pw.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/pw.json')); print('$lib', round(d['ms_per_step'],3), d['clocks'])"
done
