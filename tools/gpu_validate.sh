# round-2 validation + measurement: GPU suite, smoke, bench lines C1-C5, C4 matched T sweep
mkdir -p gpurun_out/h; rm -f gpurun_out/h/*
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/h/bench_C4.json 2> gpurun_out/h/bench_C4.err; echo benchC4=$?
for c in C3 C5 C2 C1; do timeout 600 python bench.py --config $c > gpurun_out/h/bench_$c.json 2> gpurun_out/h/bench_$c.err; echo bench$c=$?; done
for T in 8 16 32 48 64 96; do timeout 600 python bench.py --config C4 --nt 960 --T $T --steps 3 --no-e2e --no-cpu-baseline --no-other-mode --no-parity > gpurun_out/h/tsweep_C4_T$T.json 2>> gpurun_out/h/tsweep.err; echo T$T=$?; done
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/h/pytest_gpu.log 2>&1; echo pytest=$?
