# Round-end evidence: tests, smoke, bench lines for all configs, reference arm, ncu launch list + full captures (C4).
mkdir -p gpurun_out/re
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/re/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/re/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/re/bench_C4.json 2> gpurun_out/re/bench_C4.err; echo bench=$?
for c in C1 C2 C3 C5; do timeout 600 python bench.py --config $c > gpurun_out/re/bench_$c.json 2> gpurun_out/re/bench_$c.err; echo $c=$?; done
timeout 600 python bench.py --impl reference > gpurun_out/re/ref_C4.json 2>&1; echo ref=$?
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-other-mode"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/re/launches_C4.csv $CMD > gpurun_out/re/ncu_launch.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k2p -s 20 -c 1 -o gpurun_out/re/k2p_C4_fast $CMD > gpurun_out/re/ncu_full.log 2>&1; echo ncu2=$?
ncu --set full --clock-control none --import-source on -k regex:k2p -s 20 -c 1 -o gpurun_out/re/k2p_C4_matched $CMD --mode matched > gpurun_out/re/ncu_full_m.log 2>&1; echo ncu3=$?
