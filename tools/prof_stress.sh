mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 2
for wl in stress_L720_S24_H96 stress_L96_S12_H96; do
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:prnet_fwd --launch-skip 3 -c 1 -f -o gpurun_out/stress_$wl python bench.py --workload $wl --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$wl.log 2>&1
done
ls -la gpurun_out
