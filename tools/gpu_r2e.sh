# K6c (CTA-cooperative resident kernel): parity first, then the on-chip bench lines
mkdir -p gpurun_out/e
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "resident or c2_ or c5_ or c1_ or tiny or ragged or non_blocking or zero or spec or convergence" > gpurun_out/e/parity.log 2>&1; echo parity=$?
timeout 900 python -m pytest tests/test_gpu_exactness.py -q -x > gpurun_out/e/exact.log 2>&1; echo exact=$?
for c in C2 C5 C1; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/e/bench_$c.json 2> gpurun_out/e/bench_$c.err; echo bench$c=$?; done
