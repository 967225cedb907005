mkdir -p gpurun_out/f
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "resident or c2_ or c5_ or c1_ or tiny or ragged or non_blocking or zero or spec or convergence" > gpurun_out/f/parity.log 2>&1; echo parity=$?
timeout 900 python -m pytest tests/test_gpu_exactness.py -q -x > gpurun_out/f/exact.log 2>&1; echo exact=$?
for c in C2 C5; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/f/bench_$c.json 2> gpurun_out/f/bench_$c.err; echo bench$c=$?; done
HEAT1D_DEBUG=1 timeout 600 python tools/ab_time.py --variants k6cauto k6cv33 --resident True --N 1000000 --nt 1000 --cases 0.5:matched 0.5:matched:64 0.5:fast 0.5:fast:64 > gpurun_out/f/ab_c2.jsonl 2> gpurun_out/f/ab_c2.err; echo abc2=$?
HEAT1D_DEBUG=1 timeout 600 python tools/ab_time.py --variants k6cauto k6cv33 --resident True --N 1048576 --nt 20000 --cases 0.25:matched 0.25:matched:64 0.25:fast 0.25:fast:64 > gpurun_out/f/ab_c5.jsonl 2> gpurun_out/f/ab_c5.err; echo abc5=$?
