# Full evidence after the kind-4 default: GPU suite, bench lines, ncu launch list + full captures.
mkdir -p gpurun_out/r1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r1/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/r1/bench_C4.json 2> gpurun_out/r1/bench_C4.err; echo C4=$?
for c in C3 C5 C2 C1; do timeout 600 python bench.py --config $c > gpurun_out/r1/bench_$c.json 2> gpurun_out/r1/bench_$c.err; echo $c=$?; done
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-other-mode"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1/launches_C4.csv $CMD > gpurun_out/r1/ncu_launch.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k2p -s 20 -c 1 -o gpurun_out/r1/k2p_C4_fast $CMD > gpurun_out/r1/ncu_full.log 2>&1; echo ncu2=$?
ncu --set full --clock-control none --import-source on -k regex:k2p -s 20 -c 1 -o gpurun_out/r1/k2p_C4_matched $CMD --mode matched > gpurun_out/r1/ncu_full_m.log 2>&1; echo ncu3=$?
