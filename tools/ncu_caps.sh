set -u
OUT=gpurun_out/caps; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for wl in stress_L2880_S48_H96 stress_L1440_S96_H96 stress_L5760_S12_H96 electricity; do
  timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:prnet_fwd -s 2 -c 1 \
    -o $OUT/prof_$wl -f python bench.py --workload $wl --profile --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > $OUT/ncu_$wl.log 2>&1
  timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$wl.csv \
    python bench.py --workload $wl --profile --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
echo done
